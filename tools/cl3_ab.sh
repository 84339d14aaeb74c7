timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cta_group_variants or cluster_sharing" > gpurun_out/cl3_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/cl3_tests.log
SK_DEBUG_PLAN=1 timeout 120 python -c "
import torch, paper_2603_20966_b200 as sk
A=torch.empty((50000,50000),device='cuda').uniform_(-.5,.5)
for cg in (6,8):
    s=sk.Sketch(42,'gaussian',50000,256,mode='bf16',cta_group=cg); s.apply(A); torch.cuda.synchronize()
" 2>&1 | tail -4
CFGS='[["bf16","accurate",0,{"CG":6}],["bf16","accurate",0,{"CG":8}],["bf16","fast",0,{"CG":6}],["bf16","fast",0,{"CG":8}],["tf32","accurate",0,{"CG":6}],["tf32","accurate",0,{"CG":8}]]' ROUNDS=5 timeout 600 python tools/abmulti.py new 2>&1 | tail -8
