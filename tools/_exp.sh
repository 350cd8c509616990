python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -1
export EGT_BENCH_NO_VERIFY=1
for v in base mp base mp; do
  export EGT_LIB_PATH=$PWD/_variants/lib_$v.so
  echo $v $(python tools/decode_probe.py int4-2:4 2>&1 | grep plan) $(python bench.py --steps 300 --no-cpu --no-decode --no-sharded 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['dependent_chain']['ms_per_step'], {k: v['us_per_call'] for k, v in d['config']['per_shape'].items()})")
done
