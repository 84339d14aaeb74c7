# 2-GPU box: dist + virtual tests; c2 at 2 GPUs with/without graphs, with/without the overlapped core
timeout 900 python -m pytest tests/test_dist_gpu.py tests/test_virtual_gpu.py -q -p no:cacheprovider > gpurun_out/r2o_tests.log 2>&1
for lay in 2x1 1x2; do
  for g in on off; do
    timeout 600 python bench.py --gpus 2 --layout $lay --graph $g --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --no-parity > gpurun_out/r2o_c2_${lay}_g$g.json 2> gpurun_out/r2o_c2_${lay}_g$g.err
  done
done
SK_OVERLAP_CORE=0 timeout 600 python bench.py --gpus 2 --layout 1x2 --graph on --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes --no-parity > gpurun_out/r2o_c2_1x2_gon_noovl.json 2> gpurun_out/r2o_c2_1x2_gon_noovl.err
