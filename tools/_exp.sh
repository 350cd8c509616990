python -m pytest tests/test_gpu_program.py tests/test_gpu_verify.py -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
export EGT_BENCH_NO_VERIFY=1
python tools/decode_probe.py int4-2:4 2>&1 | grep plan
EGT_DECODE_NO_QKV=1 python tools/decode_probe.py int4-2:4 2>&1 | grep plan
python tools/decode_probe.py mixed-int4dense-fp16sp24 2>&1 | grep plan
python tools/decode_trace.py 8 2>&1 | head -9
