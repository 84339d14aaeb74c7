# full 1-GPU suite + smoke + default bench (round-end style)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2q_tests.log 2>&1
tail -3 gpurun_out/r2q_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2q_ref.json 2> gpurun_out/r2q_ref.err
