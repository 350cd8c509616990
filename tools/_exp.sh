bash tools/gpu_round.sh r01d > gpurun_out/round_r01d.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r01d.ncu-rep > gpurun_out/prof_r01d_summary.txt 2>&1
rm -f gpurun_out/prof_r01d.ncu-rep
