for v in _build _build_d4 _build_d5; do echo "== $v"; DJG_LIB_PATH=paper_2106_14189_b200/$v/libdjg.so timeout 300 python tools/ab_f64.py cfg3 cfg5; done
