# ncu --set full of the batch kernel on chordal-only and dense-only config-4 graphs
set -x
for w in batch_chordal batch_dense; do
  GRAPHS=16384 timeout 900 ncu --set full --clock-control none --import-source on -k regex:batch -c 1 -o gpurun_out/${TAG:-x}_$w python tools/profile_driver.py $w > gpurun_out/${TAG:-x}_$w.log 2>&1
done
ls -la gpurun_out
