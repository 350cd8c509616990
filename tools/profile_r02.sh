#!/usr/bin/env bash
# Round-2 ncu evidence (run under gpurun): the bench's M = 1 launch list with
# DRAM bytes, full captures of the M = 1 kernel, the tcgen05 many-token
# kernel (M = 80 / 272), the verify attention, and the 7B verify pass's
# per-kernel launch list; summaries written on the box.
set -uo pipefail
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:tiled_spmm -c 24 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-decode --no-sharded --no-formats > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tiled_spmm -s 10 -c 3 \
    -o $OUT/m1_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu --no-decode --no-sharded --no-formats > /dev/null 2>&1
EGT_UMMA_ALWAYS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_spmm_kernel -s 1 -c 1 \
    -o $OUT/umma80_$TAG -f python tools/umma_trace.py 4096 4096 80 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma_spmm_kernel -s 1 -c 1 \
    -o $OUT/umma272_$TAG -f python tools/umma_trace.py 11008 4096 272 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attention_tile -s 1 -c 1 \
    -o $OUT/attn272_$TAG -f python tools/verify_probe.py 272 1 > /dev/null 2>&1
for M in 80 272; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/verify${M}_launches_$TAG.csv \
      python tools/verify_probe.py $M 2 > /dev/null 2>&1
done
for f in $OUT/m1_$TAG.ncu-rep $OUT/umma80_$TAG.ncu-rep $OUT/umma272_$TAG.ncu-rep $OUT/attn272_$TAG.ncu-rep; do
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > $OUT/${b}_summary.txt 2>&1
  ncu -i $f --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
keep=[i for i,n in enumerate(h) if n in ('Kernel Name','dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active','sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed')]
for row in r[2:]:
    print({h[i]: row[i] for i in keep})" > $OUT/${b}_raw.txt
done
ls -la $OUT | tail -30
