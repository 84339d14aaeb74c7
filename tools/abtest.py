# Interleaved A/B timing of sketch configs (env knobs / ablations), min over rounds, with SM clocks.
import os, sys, json; sys.path.insert(0, '.')
import torch, paper_2603_20966_b200 as sk
try:
    import pynvml; pynvml.nvmlInit(); H = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM)
except Exception:
    clk = lambda: -1
n, r = int(os.environ.get("N", 50000)), 256
A = torch.empty((n, n), device='cuda').uniform_(-0.5, 0.5)
B = torch.empty((n, r), device='cuda')
cfgs = json.loads(sys.argv[1])  # list of {"name","mode","omega","cg","env":{},"abl":0}
res = {c["name"]: [] for c in cfgs}
clks = {c["name"]: [] for c in cfgs}
def run(c):
    for k in ("SK_A_STAGES", "SK_Y_STAGES", "SK_O_STAGES"): os.environ.pop(k, None)
    for k, v in c.get("env", {}).items(): os.environ[k] = str(v)
    s = sk.Sketch(42, 'gaussian', n, r, mode=c.get("mode", "bf16"), omega=c.get("omega", "accurate"), cta_group=c.get("cg", 0))
    s.set_ablation(c.get("abl", 0))
    s.apply(A, out=B); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(8): s.apply(A, out=B)
    e1.record(); c0 = clk(); torch.cuda.synchronize()
    res[c["name"]].append(e0.elapsed_time(e1) / 8); clks[c["name"]].append(c0)
for rnd in range(int(os.environ.get("ROUNDS", 4))):
    for c in cfgs: run(c)
for c in cfgs:
    v = sorted(res[c["name"]])
    print(f"{c['name']:28s} min {v[0]:.3f} med {v[len(v)//2]:.3f} ms  clk {clks[c['name']]}", flush=True)
