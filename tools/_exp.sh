python -m pytest tests/test_gpu_program.py tests/test_gpu_spmv.py -x -q --timeout 120 -p no:cacheprovider 2>&1 | tail -2
python tools/prog_trace.py 11008x4096:24 2>&1 | sed -n 2,6p
python tools/prog_micro.py | tail -1
python tools/prog_probe.py | tail -1 | cut -c 200-
