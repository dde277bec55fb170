# Per-phase profile of lexbfs_seg_kernel variants (tools/seg_profile_*) on the
# configuration 3 / 2 chordal graphs.
#   bash tools/seg_variants.sh variant...
python tools/dump_graph.py 32768 1024 /tmp/c3.bin
python tools/dump_graph.py 8192 8 /tmp/c2.bin
for v in "$@"; do
  for g in c3 c2; do
    echo "== $v $g"; NOPARENT=1 timeout 60 tools/seg_profile_$v /tmp/$g.bin | tail -17
  done
done
