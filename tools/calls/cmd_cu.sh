# ncu on the default c2 path after the profiled-run fallback keyed on CUDA_INJECTION64_PATH (not set by ncu: still failed)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2cu_c2_launches.csv python tools/prof_shape.py 50000 50000 256 bf16 fast gaussian 2 > gpurun_out/r2cu_c2.log 2>&1; echo "c2 prof_shape under ncu rc=$?" > gpurun_out/r2cu_rc.txt
bash tools/ncu_default.sh r2final_c2 >> gpurun_out/r2cu_rc.txt 2>&1
