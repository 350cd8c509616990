python -m pytest tests/test_gpu_verify.py tests/test_gpu_program.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -1
export EGT_BENCH_NO_VERIFY=1
python tools/decode_probe.py int4-2:4
python tools/decode_probe.py mixed-int4dense-fp16sp24
