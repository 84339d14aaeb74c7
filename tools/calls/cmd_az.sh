# epilogue-issued AllReduce of C: 2-GPU test + timing vs the fixed-order sum (2 and 4 GPUs)
timeout 900 python -m pytest tests/test_dist_gpu.py -q -p no:cacheprovider > gpurun_out/r2az_tests.log 2>&1
tail -3 gpurun_out/r2az_tests.log
for n in 2 4; do
  for ar in sum epilogue; do
    timeout 600 python bench.py --gpus $n --ar $ar --layout row --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-other-modes > gpurun_out/r2az_n${n}_$ar.json 2> gpurun_out/r2az_n${n}_$ar.err
  done
done
