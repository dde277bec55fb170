L=paper_1508_06329_b200/lib/libchordal_b200.so
for v in zero whole zero whole; do cp tools/exp/lib_$v.so $L; echo "== $v"; timeout 300 python tools/c5_time.py 2>&1 | grep -v "16384"; done
cp tools/exp/lib_whole.so $L
