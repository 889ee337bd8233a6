# A/B of Mooney-Rivlin record forms after unrolling the shared precompute loops.
export DJG_DIVS=120
echo "== T4 default (full)"; python tools/ab_models.py MR:4 MR:8 NH:4
echo "== T4 compact pipe"; DJG_FLAGS=8 python tools/ab_models.py MR:4 MR:8
echo "== T4 compact one-shot"; DJG_FLAGS=136 python tools/ab_models.py MR:4 MR:8
echo "== T4 compact pipe m3 variant"; DJG_FLAGS=8 DJG_LIB_PATH=paper_2106_14189_b200/_build_m3/libdjg.so python tools/ab_models.py MR:4 MR:8
export DJG_KIND=H8 DJG_DIVS=130
echo "== H8 default (full)"; python tools/ab_models.py MR:4 MR:8 NH:4
echo "== H8 compact"; DJG_FLAGS=8 python tools/ab_models.py MR:4 MR:8
