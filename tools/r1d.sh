python bench.py > gpurun_out/bench_r1d.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r1d.log | cut -c1-400
bash tools/ncu_default.sh r1d_c2_bf16_fast
