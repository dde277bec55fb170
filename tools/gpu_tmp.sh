timeout 300 python tools/c5_time.py
python tools/dump_csr.py 8192 8 /tmp/c2; python tools/dump_csr.py 1000000 8 /tmp/c5
for g in c2 c5; do echo == $g; timeout 60 tools/slot_profile /tmp/$g.indptr.bin /tmp/$g.indices.bin | tail -17; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "csr or seeded or config5 or linked" 2>&1 | tail -2
