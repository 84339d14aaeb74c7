#!/bin/bash
# single-GPU results sweep for BASELINE.md (JSON lines in gpurun_out/res_*.log) + ncu evidence for the default
python bench.py > gpurun_out/res_c2_n1.log 2>&1; echo "c2 n1 rc=$?"
python bench.py --workload c3 --mode tf32 --no-other-modes > gpurun_out/res_c3_n1.log 2>&1; echo "c3 rc=$?"
python bench.py --workload c4 --mode bf16 --no-other-modes > gpurun_out/res_c4_bf16.log 2>&1; echo "c4 bf16 rc=$?"
python bench.py --workload c4 --mode tf32 --omega fast --no-other-modes > gpurun_out/res_c4_tf32f.log 2>&1; echo "c4 tf32 rc=$?"
python bench.py --workload c1 --mode tf32 --omega fast --no-other-modes > gpurun_out/res_c1.log 2>&1; echo "c1 rc=$?"
bash tools/ncu_default.sh r1b_c2_bf16
