#!/usr/bin/env bash
# launch-structure experiments: empty kernel / weight stream only / full, with and without PDL
cd "${GRAFT_REPO_ROOT:-.}"
for mode in ${MODES:-1 2 0}; do
  echo "== EGT_DEBUG_MODE=$mode"
  EGT_DEBUG_MODE=$mode python tools/plan_sweep.py ${SWEEP_ARGS:-} --out gpurun_out/exp_mode$mode.json 2>&1 | python -c "
import sys, json
for line in sys.stdin:
    if line.startswith('4096') or line.startswith('11008'):
        shape, rest = line.split(' ', 1); d = json.loads(rest)
        auto = [r for r in d if r['plan'] == 'auto']
        print(shape, 'best', d[0]['plan'], d[0]['us'], 'auto', round(auto[0]['us'], 3) if auto else None)
"
done
