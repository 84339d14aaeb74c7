# in-place accumulation of split / stream-K pieces: full GPU suite, then A/B against partials + reduce
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2w_tests.log 2>&1
tail -3 gpurun_out/r2w_tests.log
for shp in "50000 50000" "12500 50000" "12500 25000" "25000 25000"; do
  for ip in 1 0 1 0; do
    echo "$shp inplace=$ip" $(SK_INPLACE=$ip python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep GB/s)
  done
done > gpurun_out/r2w_ab.txt 2>&1
for ip in 1 0; do echo "x3 inplace=$ip" $(SK_INPLACE=$ip python tools/prof_shape.py 50000 50000 256 tf32x3 accurate gaussian 3 2>&1 | grep GB/s); done >> gpurun_out/r2w_ab.txt 2>&1
for ip in 1 0; do echo "c4k1m inplace=$ip" $(SK_INPLACE=$ip python tools/prof_shape.py 2048 1000000 512 bf16 fast gaussian 3 2>&1 | grep GB/s); done >> gpurun_out/r2w_ab.txt 2>&1
