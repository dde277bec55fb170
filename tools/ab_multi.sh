# bench.py batch line for several library builds in one go: default, then each variant, twice.
L=paper_1508_06329_b200/lib/libchordal_b200.so
cp $L /tmp/lib_default.so
for round in 1 2; do
  for v in /tmp/lib_default.so "$@"; do
    cp $v $L
    python bench.py --no-secondary --no-cpu --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],3))"
  done
done
cp /tmp/lib_default.so $L
