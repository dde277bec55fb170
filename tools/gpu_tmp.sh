L=paper_1508_06329_b200/lib/libchordal_b200.so
for v in win16 win32 win16 win32; do cp tools/exp/lib_$v.so $L; echo "== $v"; timeout 300 python tools/c5_time.py 2>&1 | tail -1; done
cp tools/exp/lib_win16.so $L
