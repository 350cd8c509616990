#!/usr/bin/env bash
# One GPU measurement round (run under gpurun): GPU tests, smoke, bench, the
# ncu launch list and one full ncu capture of the SparseGemv kernel.
set -uo pipefail
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu_$TAG.txt
if [[ "${SKIP_TESTS:-0}" != 1 ]]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu_$TAG.txt 2>&1
  tail -3 $OUT/pytest_gpu_$TAG.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.txt 2>&1; tail -2 $OUT/smoke_$TAG.txt
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; tail -c 3000 $OUT/bench_$TAG.json
if [[ "${SKIP_NCU:-0}" != 1 ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:tiled_spmm -c 24 --csv --log-file $OUT/launches_$TAG.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu --no-decode --no-sharded --no-formats > /dev/null 2> $OUT/ncu_launch_$TAG.err
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tiled_spmm -s 10 -c 3 \
      -o $OUT/prof_$TAG -f python bench.py --steps 2 --warmup 1 --no-cpu --no-decode --no-sharded --no-formats > /dev/null 2> $OUT/ncu_full_$TAG.err
  ls -la $OUT/prof_$TAG.ncu-rep 2>&1 | tail -1
fi
