# Per-phase profile of the CSR slot engine on configuration 5 (tools/slot_profile*),
# plus the pivot-degree distribution of that graph.
#   bash tools/slot_variants.sh variant...     (variant "" = tools/slot_profile)
python tools/dump_csr.py 1000000 8 /tmp/c5
python - <<'PY'
import numpy as np
ip = np.fromfile("/tmp/c5.indptr.bin", np.int64)
d = np.diff(ip)
for t in (8, 16, 32, 64, 256):
    print(f"deg <= {t}: {np.mean(d <= t):.3f} of the steps")
print("max degree", d.max(), "mean", d.mean())
PY
for v in "$@"; do
  echo "== slot_profile$v"; timeout 120 tools/slot_profile$v /tmp/c5.indptr.bin /tmp/c5.indices.bin | tail -11
done
