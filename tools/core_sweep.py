# core C = Omega^T B timing over (SK_CORE_NACC, SK_CORE_STEP) for several row counts (r = 256, bf16)
import os, sys; sys.path.insert(0, '.')
import torch
import paper_2603_20966_b200 as sk
reps = 50
for mrows in (int(x) for x in os.environ.get("ROWS", "6250,12500,25000,50000").split(",")):
    B = torch.empty((mrows, 256), device='cuda').uniform_(-1, 1)
    line = []
    for nacc in ("2", "1"):
        for step in ("", "128", "256", "384", "512", "768", "1024"):
            os.environ["SK_CORE_NACC"] = nacc
            if step: os.environ["SK_CORE_STEP"] = step
            else: os.environ.pop("SK_CORE_STEP", None)
            s = sk.Sketch(42, 'gaussian', 50000, 256, mode=os.environ.get("MODE", "bf16"), omega='fast')
            C = s.core_block(B, 0); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps): s.core_block(B, 0, out=C)
                e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / reps * 1000)
            line.append(f"n{nacc}s{step or 'auto'}={sorted(ts)[1]:.1f}")
    os.environ.pop("SK_CORE_NACC", None); os.environ.pop("SK_CORE_STEP", None)
    s = sk.Sketch(42, 'gaussian', 50000, 256, mode=os.environ.get("MODE", "bf16"), omega='fast')
    C = s.core_block(B, 0); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): s.core_block(B, 0, out=C)
    e1.record(); torch.cuda.synchronize()
    print(f"m={mrows:6d} default={e0.elapsed_time(e1) / reps * 1000:.1f}us  " + " ".join(line), flush=True)
