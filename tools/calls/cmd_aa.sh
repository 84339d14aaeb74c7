# NACC = 1 (768-row units with clusters of 3 pairs) at the small per-rank shares
for shp in "6250 50000" "12500 25000" "12500 50000"; do
  for na in 2 1 2 1; do
    if [ $na = 1 ]; then E="SK_NACC=1"; else E=""; fi
    echo "$shp nacc=$na" $(env $E SK_DEBUG_PLAN=1 python tools/prof_shape.py $shp 256 bf16 fast gaussian 10 2>&1 | grep -E "plan|GB/s" | sed -e 's/.*cl=\([0-9]\) nacc=\([0-9]\).*split=\([0-9]*\) sk_len=\([0-9]*\).*grid=\([0-9]*\).*/cl=\1 nacc=\2 split=\3 sk=\4 grid=\5/' | sort -u | tr '\n' ' ')
  done
done > gpurun_out/r2aa.txt 2>&1
