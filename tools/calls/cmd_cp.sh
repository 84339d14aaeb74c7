# final 1-GPU check of the final code: GPU suite, smoke, default bench line
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2cp_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cp_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2cp_bench.json 2> gpurun_out/r2cp_bench.err
