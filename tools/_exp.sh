python -m pytest tests/test_gpu_spmv.py tests/test_gpu_verify.py -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -2
python tools/verify_probe.py 80 32; python tools/verify_probe.py 272 32
