# c4 full K: with o = 3 there is room for more A / Y stages
for rep in 1 2; do
for cfg in "" "SK_Y_STAGES=3" "SK_A_STAGES=5" "SK_A_STAGES=5 SK_Y_STAGES=3"; do
  echo "c4 [$cfg]" $(env $cfg SK_DEBUG_PLAN=1 python tools/prof_shape.py 2048 4000000 512 bf16 fast gaussian 4 2>&1 | grep -E "GB/s|plan" | sed -e 's/.*a=\([0-9]\) y=\([0-9]\) o=\([0-9]\).*smem=\([0-9]*\)/a=\1 y=\2 o=\3 smem=\4/' | sort -u | tr '\n' ' ')
done
done > gpurun_out/r2bd.txt 2>&1
