exec > gpurun_out/exp.log 2>&1
for kb in 250 125 170; do
EGT_INDEP_CTA_KB=$kb timeout 900 python bench.py --steps 50 --warmup 5 --no-decode --no-sharded 2>gpurun_out/b.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($kb, d['value'], {k: (v['us_per_call'], v['frac_of_peak']) for k,v in d['config']['formats_7b_shapes'].items()})"
done
