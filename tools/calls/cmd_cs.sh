# final ncu evidence of the default c2 line (launch list + full capture of the sketch kernel)
bash tools/ncu_default.sh r2final_c2
