timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2bh_tests.log 2>&1
tail -2 gpurun_out/r2bh_tests.log
Q="python tools/prof_shape.py 50000 50000 256 tf32x3 accurate gaussian 3"
$Q > gpurun_out/r2bh_x3.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sketch_gemm -s 1 -c 1 $Q > gpurun_out/r2bh_ncu.log 2>&1
python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 10 >> gpurun_out/r2bh_x3.log 2>&1
