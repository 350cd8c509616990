python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
for v in zp cur zp cur; do
  if [ $v = zp ]; then export EGT_LIB_PATH=$PWD/_variants/lib_zp.so; else unset EGT_LIB_PATH; fi
  python bench.py --steps 500 --no-cpu --no-decode --no-sharded 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['config']['per_shape']['4096x4096']['us_per_call'], d['config']['per_shape']['11008x4096']['us_per_call'], d['config']['per_shape']['4096x11008']['us_per_call'], (d['clocks'] or {}).get('sm_mhz'))"
done
