# counting-signal device barrier (new default) vs the symmetric-memory handle barrier: dist tests, phase timeline, bench A/B at 4 GPUs
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x > gpurun_out/r2ch_dist_tests.txt 2>&1 || { tail -30 gpurun_out/r2ch_dist_tests.txt; exit 1; }
for spec in 2x2 4x1; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/dist_phases.py $spec >> gpurun_out/r2ch_phases.txt 2>&1; done
SK_NVLS_MIN=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/dist_phases.py 2x2 >> gpurun_out/r2ch_phases_nvls2.txt 2>&1
for rep in 1 2; do
  timeout 900 python bench.py --gpus 4 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2ch_bench_n4_new$rep.json 2> gpurun_out/r2ch_bench_n4_new$rep.err
  SK_TORCH_BARRIER=1 timeout 900 python bench.py --gpus 4 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2ch_bench_n4_torch$rep.json 2> gpurun_out/r2ch_bench_n4_torch$rep.err
done
timeout 900 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2ch_bench_n2_new.json 2> gpurun_out/r2ch_bench_n2_new.err
SK_TORCH_BARRIER=1 timeout 900 python bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-other-modes > gpurun_out/r2ch_bench_n2_torch.json 2> gpurun_out/r2ch_bench_n2_torch.err
