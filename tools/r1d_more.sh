bash tools/ncu_default.sh r1d_c3_tf32_accurate --workload c3 --mode tf32
bash tools/ncu_default.sh r1d_c4_bf16_fast --workload c4
