# remainder launch: tests + per-rank shares with / without it
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "ragged_row_remainder or streamk_inplace or sketch_parity or integer_exact" > gpurun_out/r2x_tests.log 2>&1
tail -3 gpurun_out/r2x_tests.log
for shp in "6250 50000" "12500 25000" "12500 50000" "50000 50000"; do
  for nr in 0 1 0 1; do
    if [ $nr = 1 ]; then E="SK_NO_REMAINDER=1"; else E=""; fi
    echo "$shp no_remainder=$nr" $(env $E python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep GB/s)
  done
done > gpurun_out/r2x_ab.txt 2>&1
