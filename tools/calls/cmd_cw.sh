# ncu on the default c2 path with the profiler detected by NV_COMPUTE_PROFILER_PERFWORKS_DIR, then the final ncu evidence
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2cw_c2_launches.csv python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 2 > gpurun_out/r2cw_c2.log 2>&1; echo "c2 prof_shape under ncu rc=$?" > gpurun_out/r2cw_rc.txt
bash tools/ncu_default.sh r2final_c2 >> gpurun_out/r2cw_rc.txt 2>&1
