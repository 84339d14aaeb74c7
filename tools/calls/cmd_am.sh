# remaining 1-GPU workload lines: c1 (launch-latency bound) and c3 (row-block, Rademacher), c4
for wl in c1 c3 c4; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-e2e --no-other-modes > gpurun_out/r2am_$wl.json 2> gpurun_out/r2am_$wl.err
done
