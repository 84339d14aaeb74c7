# ncu of the final c4 (full size) and c3 sketch kernels, with launch lists of their bench steps
for wl in c4 c3; do
  B="python bench.py --workload $wl --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity"
  $B > gpurun_out/r2bf_plain_$wl.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2bf_launch_$wl.csv $B > gpurun_out/r2bf_ncu1_$wl.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 3 -c 1 -o gpurun_out/r2bf_$wl -f $B > gpurun_out/r2bf_ncu2_$wl.log 2>&1
done
