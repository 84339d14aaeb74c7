#!/bin/bash
# ncu --set full of one sketch_gemm launch: tools/ncu_one.sh <tag> [bench args]
tag=$1; shift
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-other-modes $@"
$CMD > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sketch_gemm -s 3 -c 1 -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?"
