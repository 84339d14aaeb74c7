for shp in "12500 50000" "6250 50000" "16384 50000" "25000 25000" "50000 50000"; do
  set -- $shp
  timeout 300 python tools/clab.py $1 $2 256 bf16 fast 0,6,8
done
timeout 300 python tools/clab.py 12500 50000 256 bf16 accurate 6,8
