timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "csr or seeded or config5" 2>&1 | tail -3
timeout 300 python tools/sanitize_driver.py slot
timeout 300 python tools/c5_time.py
