# small n1 (short-wide, few rows): plan and time; remainder-launch A/B
for n1 in 106 128 256 512 1024; do
  echo "$n1" $(SK_DEBUG_PLAN=1 python tools/prof_shape.py $n1 50000 256 bf16 fast gaussian 10 2>&1 | grep -E "plan|GB/s" | sort -u | tr '\n' ' ')
done > gpurun_out/r2y_small.txt 2>&1
for shp in "6250 50000" "12500 25000"; do
  for nr in 0 1 0 1; do
    if [ $nr = 1 ]; then E="SK_NO_REMAINDER=1"; else E=""; fi
    echo "$shp no_remainder=$nr" $(env $E python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep GB/s)
  done
done >> gpurun_out/r2y_small.txt 2>&1
