# Bounds-checked slot engine on one B200 (stands in for compute-sanitizer memcheck,
# which this pool no longer runs).
#   here:   bash tools/ab_variants.sh build bounds "-DCHORDAL_SLOT_BOUNDS"   (-> tools/exp/bounds.so)
#   on GPU: bash tools/bounds_check.sh TAG
# Every subscript / pointer offset of the slot state (slot_engine.cuh, ChkPtr) traps
# with the array's name when it leaves its array.  Runs the sanitizer driver's slot
# part (all-shared-memory, shared-ids and global-state kernels, seeded / descending
# arbitration), the GPU parity tests that reach the slot engine, and configuration 5
# (CSR n = 10^6) plus the CSR n = 8192 timing inputs, then restores the product library.
TAG=${1:-r02_bounds}
L=paper_1508_06329_b200/lib/libchordal_b200.so
O=gpurun_out/${TAG}_slot_bounds.txt
cp $L /tmp/lib_product.so
cp tools/exp/bounds.so $L
strings $L | grep -c "slot bounds" > $O
echo "== sanitize_driver slot" >> $O
timeout 600 python tools/sanitize_driver.py slot >> $O 2>&1; echo "rc=$?" >> $O
echo "== pytest -m gpu -k 'csr or slot or seeded or arb or chordal_random or left'" >> $O
timeout 900 python -m pytest tests -m gpu -q -k "csr or slot or seeded or arb or chordal_random or left" 2>&1 | tail -4 >> $O
echo "== tools/c5_time.py (config 5 + CSR n = 8192)" >> $O
timeout 600 python tools/c5_time.py >> $O 2>&1; echo "rc=$?" >> $O
cp /tmp/lib_product.so $L
cat $O
