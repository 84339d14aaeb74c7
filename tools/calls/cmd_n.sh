# per-rank shapes of c2 at 8 GPUs (4x2, 8x1, 2x4) and 4 GPUs (2x2, 4x1): cluster size sweep, bf16 / fast
for shp in "12500 25000" "6250 50000" "25000 12500" "25000 25000" "12500 50000"; do
  for cg in 0 4 6 8; do
    echo "$shp CG=$cg" $(CG=$cg SK_DEBUG_PLAN=1 python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep -E "plan|GB/s" | sed -e 's/.*cl=\([0-9]\).*split=\([0-9]*\) sk_len=\([0-9]*\).*grid=\([0-9]*\).*/cl=\1 split=\2 sk=\3 grid=\4/' | sort -u | tr '\n' ' ')
  done
done > gpurun_out/r2n_shares.txt 2>&1
