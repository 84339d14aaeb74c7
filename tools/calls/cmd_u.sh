# c2 ring splits with a deeper Omega ring (the trace shows the Omega sharing chain on the critical path)
Q="python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 5"
for cfg in "" "SK_Y_STAGES=1 SK_O_STAGES=8" "SK_A_STAGES=2 SK_O_STAGES=8" "SK_A_STAGES=2 SK_Y_STAGES=1 SK_O_STAGES=8" ""; do
  echo "c2 [$cfg]" $(env $cfg SK_DEBUG_PLAN=1 $Q 2>&1 | grep -E "plan|GB/s" | sed -e 's/.*a=\([0-9]\) y=\([0-9]\) o=\([0-9]\).*grid=\([0-9]*\).*/a=\1 y=\2 o=\3 grid=\4/' | sort -u | tr '\n' ' ')
done > gpurun_out/r2u_sweep.txt 2>&1
