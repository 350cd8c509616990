#!/usr/bin/env bash
# ncu captures for profiles/ (run under gpurun): full sets of the M=1
# SparseGemv under its dependent (full-chip) plans, the many-token kernel,
# and the decode-step kernels.
set -uo pipefail
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r01}
for sh in 4096x4096 11008x4096 4096x11008; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:tiled_spmm -s 3 -c 1 \
      -o $OUT/dep_${sh}_$TAG -f python tools/prof_one.py --shape $sh --launches 5 > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wide_spmm -s 2 -c 1 \
    -o $OUT/wide_$TAG -f python tools/verify_probe.py 80 1 > /dev/null 2>&1
ls -la $OUT/*_$TAG.ncu-rep
# summaries on the box (the full reports are too large to bring back)
for f in $OUT/dep_*_$TAG.ncu-rep $OUT/wide_$TAG.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > $OUT/${b}_summary.txt 2>&1
  k=tiled_spmm; o=paper_2605_11582_b200/_lib/obj/spmm_tiled.cu.o
  case $b in wide_*) k=wide_spmm; o=paper_2605_11582_b200/_lib/obj/spmm_wide.cu.o;; esac
  python tools/ncu_lines.py $f $o $k 25 > $OUT/${b}_lines.txt 2>&1
  ncu -i $f --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
keep=[i for i,n in enumerate(h) if n in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active','smsp__inst_executed_pipe_tensor_op_hmma.sum')]
print({h[i]: (v[i], r[1][i]) for i in keep})" > $OUT/${b}_raw.txt
  rm -f $f
done
ls -la $OUT
