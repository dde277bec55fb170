timeout 300 python tools/c5_time.py
