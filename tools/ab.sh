timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for v in _build _build_q6s8 _build_q7s4 _build_q5s4; do echo "== $v"; DJG_LIB_PATH=paper_2106_14189_b200/$v/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg5; done
