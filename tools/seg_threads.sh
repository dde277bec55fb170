# CTA-engine thread-count sweep on the configuration 2 / 3 graphs (tools/seg_time).
python tools/dump_graph.py 32768 1024 /tmp/c3.bin
python tools/dump_graph.py 32768 0.5 /tmp/c3d.bin
python tools/dump_graph.py 8192 8 /tmp/c2.bin
python tools/dump_graph.py 8192 0.5 /tmp/c2d.bin
for g in c3 c3d c2 c2d; do
  for t in 256 512 1024; do SEG_THREADS=$t timeout 60 tools/seg_time /tmp/$g.bin; done
  timeout 60 tools/seg_time /tmp/$g.bin
done
