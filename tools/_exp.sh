exec > gpurun_out/exp.log 2>&1; set -x
for m in 0 14; do EGT_DEBUG_MODE=$m timeout 300 python tools/peer_probe.py; done
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -m gpu 2>&1 | tail -3
EGT_DEBUG_MODE=14 timeout 900 python -m pytest tests/test_gpu_peer.py -x -q -m gpu 2>&1 | tail -3
