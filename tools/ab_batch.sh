# A/B of the batch kernel: the in-tree library vs a variant build of it (same API),
# bench.py batch line only.  Build the variant here first, e.g.
#   CHORDAL_NVCC_EXTRA="-DSOME_FLAG=1" python -c "import __graft_entry__ as g; g.build()"   (after touching a source)
#   cp paper_1508_06329_b200/lib/libchordal_b200.so tools/exp/lib_variant.so; rebuild the default
#   bash tools/ab_batch.sh tools/exp/lib_variant.so
L=paper_1508_06329_b200/lib/libchordal_b200.so
V=${1:-tools/exp/lib_variant.so}
cp $L /tmp/lib_default.so
for v in default variant default variant; do
  if [ $v = variant ]; then cp $V $L; else cp /tmp/lib_default.so $L; fi
  python bench.py --no-secondary --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3))"
done
cp /tmp/lib_default.so $L
