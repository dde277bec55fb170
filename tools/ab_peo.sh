# A/B of the PEO lines (peo_ms) of bench.py's single-graph section: in-tree library vs a variant.
L=paper_1508_06329_b200/lib/libchordal_b200.so
V=${1:-tools/exp/lib_variant.so}
cp $L /tmp/lib_default.so
for v in default variant default variant; do
  if [ $v = variant ]; then cp $V $L; else cp /tmp/lib_default.so $L; fi
  python bench.py --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); sg=d['single_graph']
print('$v', ' '.join(f\"{k}={sg[k]['peo_ms']:.4f}/{sg[k].get('peo_parent_search_ms') or 0:.4f}\" for k in sg if isinstance(sg[k], dict) and 'peo_ms' in sg[k]))"
done
cp /tmp/lib_default.so $L
