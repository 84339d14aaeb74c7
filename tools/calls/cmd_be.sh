# c2 ring split with 8 producer warps, interleaved x2
for rep in 1 2; do
for cfg in "" "SK_A_STAGES=4" "SK_O_STAGES=3" "SK_A_STAGES=2 SK_O_STAGES=8"; do
  echo "c2 [$cfg]" $(env $cfg SK_DEBUG_PLAN=1 python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 8 2>&1 | grep -E "GB/s|plan" | sed -e 's/.*a=\([0-9]\) y=\([0-9]\) o=\([0-9]\).*smem=\([0-9]*\)/a=\1 y=\2 o=\3 smem=\4/' | sort -u | tr '\n' ' ')
done
done > gpurun_out/r2be.txt 2>&1
