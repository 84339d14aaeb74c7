# final-state check on a 2-GPU box: whole GPU suite (multi-GPU tests included), smoke, default bench,
# launch list + ncu --set full of the default bench's sketch kernel
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2ac_tests.log 2>&1
tail -3 gpurun_out/r2ac_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ac_smoke.log 2>&1
B="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-other-modes --no-parity"
timeout 600 python bench.py > gpurun_out/r2ac_bench.json 2> gpurun_out/r2ac_bench.err
$B > gpurun_out/r2ac_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ac_launch_c2.csv $B > gpurun_out/r2ac_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 4 -c 1 -o gpurun_out/r2ac_c2 -f $B > gpurun_out/r2ac_ncu2.log 2>&1
