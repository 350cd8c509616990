export EGT_BENCH_NO_VERIFY=1
for v in t900 t2500; do
  export EGT_LIB_PATH=$PWD/_variants/lib_$v.so
  echo $v $(python tools/decode_probe.py int4-2:4 2>&1 | grep plan) $(python tools/decode_probe.py mixed-int4dense-fp16sp24 2>&1 | grep plan)
  python bench.py --steps 300 --no-cpu --no-decode --no-sharded 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['config']['dependent_chain'])"
done
