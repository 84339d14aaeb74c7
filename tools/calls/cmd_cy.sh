# last rehearsal of the final code (templated peer sum, profiler-safe path): GPU suite, smoke, bench N = 1 / 2 / 4, reference arm
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2cy_tests.log 2>&1
tail -3 gpurun_out/r2cy_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cy_smoke.log 2>&1
for n in 1 2 4; do timeout 900 python bench.py --gpus $n > gpurun_out/r2cy_bench_n$n.json 2> gpurun_out/r2cy_bench_n$n.err; done
timeout 600 python bench.py --impl reference > gpurun_out/r2cy_ref.json 2> gpurun_out/r2cy_ref.err
