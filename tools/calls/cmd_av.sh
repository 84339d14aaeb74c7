# final-state check on a 2-GPU box: whole GPU suite, smoke, default bench, 2-GPU bench
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2av_tests.log 2>&1
tail -3 gpurun_out/r2av_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2av_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2av_bench.json 2> gpurun_out/r2av_bench.err
timeout 600 python bench.py --gpus 2 > gpurun_out/r2av_bench_n2.json 2> gpurun_out/r2av_bench_n2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2av_ref.json 2> gpurun_out/r2av_ref.err
