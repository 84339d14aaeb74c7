# final code: GPU suite on one GPU, smoke, smoke under ncu (launch list)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2cx_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cx_smoke.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2cx_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cx_smoke_ncu.log 2>&1; echo "smoke under ncu rc=$?" >> gpurun_out/r2cx_smoke.log
