# A/B of library builds on the hot workloads (tools/variant_time.py).
#   here:   bash tools/ab_variants.sh build NAME "nvcc flags"   (-> tools/exp/NAME.so)
#   on GPU: bash tools/ab_variants.sh run "workloads" NAME...   (alternates the builds twice)
set -e
L=paper_1508_06329_b200/lib/libchordal_b200.so
if [ "$1" = build ]; then
  mkdir -p tools/exp
  CHORDAL_NVCC_EXTRA="$3" python -c "
import sys; sys.path.insert(0, 'paper_1508_06329_b200'); import _build; _build.build(force=True)" >/dev/null
  cp $L tools/exp/$2.so
  exit 0
fi
W="$2"; shift 2
cp $L /tmp/lib_inplace.so
rm -f /tmp/variant_hashes.json
for rep in 1 2; do
  for v in "$@"; do
    cp tools/exp/$v.so $L
    echo "== $v (pass $rep)"
    timeout 900 python tools/variant_time.py $W || echo "FAILED $v"
  done
done
cp /tmp/lib_inplace.so $L
