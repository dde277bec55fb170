timeout 900 python -m pytest tests/test_gpu_abi_edges.py tests/test_gpu_parity.py -m gpu -q -x -k "host or padded or reference_graph or batch" 2>&1 | tail -3
