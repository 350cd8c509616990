bash tools/gpu_round.sh r01c > gpurun_out/round_r01c.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r01c.ncu-rep > gpurun_out/prof_r01c_summary.txt 2>&1
ncu -i gpurun_out/prof_r01c.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=[i for i,n in enumerate(h) if n in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','launch__grid_size','dram__throughput.avg.pct_of_peak_sustained_elapsed')]
for v in r[2:]: print({h[i]: v[i] for i in keep})" > gpurun_out/prof_r01c_raw.txt
rm -f gpurun_out/prof_r01c.ncu-rep
