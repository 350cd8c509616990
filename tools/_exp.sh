python -m pytest tests/test_gpu_program.py -x -q --timeout 120 -p no:cacheprovider 2>&1 | tail -2
python tools/prog_trace.py chain:4 2>&1 | sed -n 1,30p
python tools/prog_probe.py | tail -1 | cut -c 200-
