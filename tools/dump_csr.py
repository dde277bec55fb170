"""Write a CSR graph for tools/slot_profile: configuration 5 (gen_chordal_random(N, K, 0)
drawn on the GPU) as int64 indptr + int32 indices files.

    python tools/dump_csr.py N K out_prefix
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1508_06329_b200.generate import gen_chordal_random_csr_device  # noqa: E402


def main(n, k, out):
    ip, ix = gen_chordal_random_csr_device(n, k, 0)
    ip.cpu().numpy().tofile(out + ".indptr.bin")
    ix.cpu().numpy().tofile(out + ".indices.bin")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3])
