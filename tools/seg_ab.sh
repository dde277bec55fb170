# A/B of two tools/seg_time builds on the configuration 2 / 3 graphs.
#   bash tools/seg_ab.sh tools/seg_time tools/seg_time_variant
python tools/dump_graph.py 32768 1024 /tmp/c3.bin
python tools/dump_graph.py 32768 0.5 /tmp/c3d.bin
python tools/dump_graph.py 8192 8 /tmp/c2.bin
python tools/dump_graph.py 8192 0.5 /tmp/c2d.bin
for round in 1 2; do
  for g in c3 c3d c2 c2d; do
    for b in "$@"; do echo -n "$b: "; timeout 60 $b /tmp/$g.bin; done
  done
done
