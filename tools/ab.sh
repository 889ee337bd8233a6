timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/probe_perf.py cfg1 cfg2 cfg3 cfg4 cfg5 2>&1 | cut -c1-200
