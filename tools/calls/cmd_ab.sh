# in-place piece limit at the 8-GPU row share and c2 full (stream-K / split-K piece counts 6 and 2)
for shp in "6250 50000" "6250 25000" "50000 50000"; do
  for mx in 4 8 4 8; do
    echo "$shp inplace_max=$mx" $(SK_INPLACE_MAX=$mx python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep GB/s)
  done
done > gpurun_out/r2ab.txt 2>&1
