# c4 full K: ring split a=3,o=4 (planner) vs a=4,o=3 vs o=3, interleaved x3
for rep in 1 2 3; do
for cfg in "" "SK_A_STAGES=4 SK_O_STAGES=3" "SK_O_STAGES=3"; do
  echo "c4 [$cfg]" $(env $cfg python tools/prof_shape.py 2048 4000000 512 bf16 fast gaussian 4 2>&1 | grep GB/s)
done
done > gpurun_out/r2bb.txt 2>&1
