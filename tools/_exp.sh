exec > gpurun_out/exp.log 2>&1
timeout 900 python -m pytest tests/test_gpu_compress.py -x -q -m gpu 2>&1 | tail -15
