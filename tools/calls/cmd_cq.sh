# final sanity of the other workloads' bench lines on 1 GPU (c1, c3, c4)
for w in c1 c3 c4; do timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-other-modes > gpurun_out/r2cq_$w.json 2> gpurun_out/r2cq_$w.err; done
