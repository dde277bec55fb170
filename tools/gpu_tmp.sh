timeout 300 python tools/engine_time.py 8192 8
timeout 300 python tools/engine_time.py 4096 4
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
