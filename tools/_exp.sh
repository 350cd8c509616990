exec > gpurun_out/exp.log 2>&1
for st in 300 1000 300 3000; do
timeout 600 python bench.py --steps $st --warmup 10 --no-decode --no-sharded --no-formats 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($st, d['value'], d['roofline']['frac'], d['clocks'])"
done
