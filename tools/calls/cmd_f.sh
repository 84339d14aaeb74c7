# c4-shape ring-depth sweep (single pass, NCOL = 2)
P="python tools/prof_shape.py 2048 1000000 512 bf16 fast gaussian 5"
for cfg in "" "SK_A_STAGES=2" "SK_A_STAGES=2 SK_Y_STAGES=1" "SK_NCOL_CL=4" "SK_NCOL_CL=4 SK_A_STAGES=2" "SK_PREFETCH=4" "SK_NCOL=1"; do
  echo "[$cfg]" $(env $cfg SK_DEBUG_PLAN=1 $P 2>&1 | grep -E "plan|GB/s" | sed -e 's/.*a=\([0-9]\) y=\([0-9]\) o=\([0-9]\).*grid=\([0-9]*\).*/a=\1 y=\2 o=\3 grid=\4/' | sort -u | tr '\n' ' ')
done > gpurun_out/r2f_sweep.txt 2>&1
