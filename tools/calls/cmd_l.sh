# launch lists (ncu gpu__time_duration) of the bench steps: c2 bf16 default, c2 tf32x3, c4; ncu --set full of the x3 sketch
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity"
$B > gpurun_out/r2l_plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launch_c2.csv $B > gpurun_out/r2l_ncu1.log 2>&1
$B --mode tf32x3 > gpurun_out/r2l_plain_x3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launch_x3.csv $B --mode tf32x3 > gpurun_out/r2l_ncu2.log 2>&1
$B --workload c4 > gpurun_out/r2l_plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2l_launch_c4.csv $B --workload c4 > gpurun_out/r2l_ncu3.log 2>&1
Q="python tools/prof_shape.py 50000 50000 256 tf32x3 accurate gaussian 2"
$Q > gpurun_out/r2l_x3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 1 -c 1 -o gpurun_out/r2l_x3 -f $Q > gpurun_out/r2l_ncu4.log 2>&1
