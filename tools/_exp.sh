exec > gpurun_out/exp.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 300 python tools/verify_probe.py 2>&1 | tail -3
EGT_DENSE_TREE_MASK=1 timeout 300 python tools/verify_probe.py 2>&1 | tail -3
