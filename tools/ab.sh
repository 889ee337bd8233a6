timeout 300 python tools/ab_exp.py cfg3 cfg5
DJG_FLAGS=128 timeout 300 python tools/ab_exp.py cfg3 cfg5
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tled.py tests/test_gpu_multipart.py -x -q 2>&1 | tail -3
