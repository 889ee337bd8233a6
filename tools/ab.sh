timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "device_layout" 2>&1 | tail -15
./tests/cpp/_build/test_dropin 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_dropin_cpp.py -q 2>&1 | tail -2
