python -m pytest tests/test_gpu_verify.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -1
export EGT_BENCH_NO_VERIFY=1
python tools/decode_probe.py int4-2:4 2>&1 | grep -v Warn
python tools/decode_probe.py int4-2:4 2>&1 | grep -v Warn
