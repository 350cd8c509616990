python -m pytest tests/test_gpu_program.py tests/test_gpu_spmv.py -x -q --timeout 120 -p no:cacheprovider 2>&1 | tail -2
python tools/prog_trace.py 11008x4096:24 2>&1 | sed -n 2,6p
python tools/prog_micro.py | tail -1
python tools/prog_probe.py | tail -1 | cut -c 200-
python bench.py --steps 300 --no-sharded 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['config']['per_shape'], d['config']['dependent_chain'], d['cpu_baseline']['parity_max_rel_err_vs_gpu'])"
