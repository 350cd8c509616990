python -m pytest tests/test_gpu_spmv.py -q -k "many or wide" --timeout 120 -p no:cacheprovider 2>&1 | tail -1
for M in 80 272; do echo $(python tools/verify_probe.py $M 32 2>&1 | grep M=); done
