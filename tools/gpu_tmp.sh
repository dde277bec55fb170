timeout 300 python tools/c5_time.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_left.py -m gpu -q -x -k "csr or seeded or config5 or linked or left" 2>&1 | tail -2
