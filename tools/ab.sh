for v in _build_o1 _build_o5; do echo "== $v TLED"; DJG_FLAGS=64 DJG_LIB_PATH=paper_2106_14189_b200/$v/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg5; done
echo "== TLED nopipe"; DJG_FLAGS=192 DJG_LIB_PATH=paper_2106_14189_b200/_build_o1/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg5
for v in _build_o1 _build_o4; do echo "== $v H8 compact"; DJG_FLAGS=8 DJG_LIB_PATH=paper_2106_14189_b200/$v/libdjg.so timeout 300 python tools/ab_exp.py cfg4; done
echo "== H8 compact nopipe"; DJG_FLAGS=136 DJG_LIB_PATH=paper_2106_14189_b200/_build_o1/libdjg.so timeout 300 python tools/ab_exp.py cfg4
echo "== H8 full (default)"; DJG_LIB_PATH=paper_2106_14189_b200/_build_o1/libdjg.so timeout 300 python tools/ab_exp.py cfg4
echo "== T4 full"; DJG_FLAGS=32 DJG_LIB_PATH=paper_2106_14189_b200/_build_o1/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg5
echo "== T4 full nopipe"; DJG_FLAGS=160 DJG_LIB_PATH=paper_2106_14189_b200/_build_o1/libdjg.so timeout 300 python tools/ab_exp.py cfg3 cfg5
