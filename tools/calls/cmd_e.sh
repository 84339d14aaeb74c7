# ncu --set full of the c4-shaped (single pass, 16-CTA clusters) and c2 sketch kernels
P="python tools/prof_shape.py 2048 1000000 512 bf16 fast gaussian 2"
Q="python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 2"
$P > gpurun_out/r2e_c4.log 2>&1 && $Q > gpurun_out/r2e_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 1 -c 1 -o gpurun_out/r2e_c4 -f $P > gpurun_out/r2e_ncu_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 1 -c 1 -o gpurun_out/r2e_c2 -f $Q > gpurun_out/r2e_ncu_c2.log 2>&1
