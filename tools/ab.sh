for v in _build _build_r12; do echo "== $v"; DJG_LIB_PATH=paper_2106_14189_b200/$v/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg4 cfg5; done
