# tf32x3 with evict-last output rows: parity + DRAM traffic (ncu) + time
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "tf32x3" > gpurun_out/r2bg_tests.log 2>&1
tail -2 gpurun_out/r2bg_tests.log
Q="python tools/prof_shape.py 50000 50000 256 tf32x3 accurate gaussian 3"
$Q > gpurun_out/r2bg_x3.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sketch_gemm -s 1 -c 1 $Q > gpurun_out/r2bg_ncu.log 2>&1
