# c4 ring split, interleaved repeats (K = 1e6 shape and full K = 4e6)
for rep in 1 2 3; do
for cfg in "" "SK_A_STAGES=4 SK_O_STAGES=3" "SK_O_STAGES=3"; do
  echo "c4k1m [$cfg]" $(env $cfg python tools/prof_shape.py 2048 1000000 512 bf16 fast gaussian 10 2>&1 | grep GB/s)
done
done > gpurun_out/r2ae.txt 2>&1
for cfg in "" "SK_A_STAGES=4 SK_O_STAGES=3"; do
  echo "c4 full [$cfg]" $(env $cfg python tools/prof_shape.py 2048 4000000 512 bf16 fast gaussian 5 2>&1 | grep GB/s)
done >> gpurun_out/r2ae.txt 2>&1
