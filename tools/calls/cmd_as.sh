timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2as_tests.log 2>&1
tail -3 gpurun_out/r2as_tests.log
for shp in "50000 50000" "25000 25000" "12500 25000"; do
  for ip in 1 0; do echo "$shp inplace=$ip" $(SK_INPLACE=$ip python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep GB/s); done
done > gpurun_out/r2as_ab.txt 2>&1
