python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -4
timeout 300 python tools/_repro_fmt.py 2>&1 | grep -v Warn | tail -9
