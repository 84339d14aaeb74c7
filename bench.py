#!/usr/bin/env python
"""bench.py -- the sketch B = A*Omega + Nystrom core C = Omega^T*B on B200 (BASELINE.json metric).

Default workload (N = 1): BASELINE.json configs[1] = c2, the Nystrom core of a symmetric PSD
n = 50,000 matrix (synthetic RBF kernel of X ~ U[0,1)^{50000 x 3072}, the CIFAR-10-shaped
analogue of PAPER.md:1013-1024), r = 256 Gaussian Omega regenerated in-kernel.  One step = one
full pass of the hot path: B = A Omega (fused Omega tiles + tcgen05 GEMM [+ split-K reduce]) and
C = Omega^T B (Omega regenerated) [+ AllReduce of C for N > 1].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--mode tf32]
  torchrun --nproc-per-node N bench.py --gpus N ...      (row-block layout by default)
  python bench.py --impl reference ...                    (the fp64 CPU oracle on host cores)

Prints ONE JSON line (rank 0).  value = effective GB/s of A over the whole job (all ranks' A
bytes / max-over-ranks device time); TFLOP/s, per-phase device times, roofline of the dominant
kernel, the oracle baseline, e2e (host buffers), clocks and launch counts ride along.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch A·Ω effective HBM GB/s + TFLOP/s (% roofline) at 1/2/4/8 B200; Nyström core time"

WORKLOADS = {
    "c1": dict(desc="c1: A 512x512 symmetric fp32, Gaussian Omega r=16, B=A*Omega and C=Omega^T*B",
               n1=512, n2=512, r=16, dist="gaussian", nystrom=True, a="symuniform"),
    "c2": dict(desc="c2: Nystrom core, symmetric PSD A n=50,000 (RBF kernel of X~U[0,1)^{50000x3072}), "
                    "r=256 Gaussian",
               n1=50000, n2=50000, r=256, dist="gaussian", nystrom=True, a="rbf", d=3072),
    "c3": dict(desc="c3: tall-skinny A 4,000,000x2,048 fp32 U[-1/2,1/2), r=128 Rademacher, row-block",
               n1=4_000_000, n2=2048, r=128, dist="rademacher", nystrom=False, a="uniform"),
    "c4": dict(desc="c4: short-wide A 2,048x4,000,000 fp32 U[-1/2,1/2), r=512 Gaussian",
               n1=2048, n2=4_000_000, r=512, dist="gaussian", nystrom=False, a="uniform"),
    "c5": dict(desc="c5: large symmetric PSD A n=200,000 (RBF kernel of X~U[0,1)^{200000x64}; 160 GB, "
                    "for 8 GPUs), Nystrom r=1,024, 2D grid, AllReduce of C",
               n1=200_000, n2=200_000, r=1024, dist="gaussian", nystrom=True, a="rbf", d=64),
}

SEED_OMEGA = 42
SEED_A = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}
NOMINAL_TF32_OVER_BF16 = 1.1 / 2.25  # B200 dense tensor peaks (B200_PROFILING.md nominal table)


def auto_layout(wl_name, world):
    """The processor grid BASELINE.json's configs name: c2 ("2/4/8 with 2D grid") and c5 ("2D grid"): the
    most square p1 x p2 grid with p1 >= p2 (2x1, 2x2, 4x2); c3 row-block (zero communication); c4
    column-block (reduce-scatter of B).  The grid the paper's own selection rule picks for P <= n1
    (sec. 4.3 Case 1: P x 1, zero words for B) is `--layout row` (measured faster
    at 4 GPUs: 0.552 vs 0.564 ms)."""
    if world == 1:
        return "row"
    if wl_name == "c4":
        return "col"
    if wl_name in ("c2", "c5"):
        p2 = 1
        for d in range(1, int(world ** 0.5) + 1):
            if world % d == 0:
                p2 = d
        return f"{world // p2}x{p2}"
    return "row"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# The JSON line is the only thing on stdout: everything else written to file descriptor 1 while
# the bench runs -- NCCL's version banner, library prints -- is sent to stderr.
_JSON_FD = None


def _stdout_to_stderr():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(obj):
    sys.stdout.flush()
    os.write(_JSON_FD if _JSON_FD is not None else 1, (json.dumps(obj) + "\n").encode())


SPEC = {"hbm": 7700.0, "bf16": 2250.0, "tf32": 1100.0}  # nominal B200 (B200_PROFILING.md table): context only


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        pk = dict(hbm=float(p["hbm_gbs"]), bf16=float(p["bf16_tflops"]),
                  bf16_sus=float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                  source="MEASURED_PEAKS.json (measured)")
    else:
        pk = dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="B200_PROFILING.md fallback")
    # TF32: cuBLAS TF32 8192^3 measured on this pool (tools/measure_tf32_peak.py), else bf16 x nominal ratio
    tp = os.path.join(ROOT, "profiles", "tf32_peak.json")
    if os.path.exists(tp):
        with open(tp) as f:
            pk["tf32"] = float(json.load(f)["tf32_tflops"])
        pk["tf32_source"] = "profiles/tf32_peak.json (cuBLAS TF32 8192^3, measured)"
    else:
        pk["tf32"] = pk["bf16"] * NOMINAL_TF32_OVER_BF16
        pk["tf32_source"] = "bf16 measured x 1.1/2.25 nominal"
    return pk


def roofline(mode, kern_bytes, kern_flops, kern_s, peaks):
    """Roofline of the sketch kernel for one step's launches: the binding resource is whichever of HBM
    (algorithmic bytes / measured copy bandwidth) and the tensor pipe (flops / the measured peak of the
    mode's MMA: bf16; tf32; tf32x3 = tf32 / 3, three MMAs per product) takes longer at its peak."""
    tc_peak = {"bf16": peaks["bf16"], "tf32": peaks["tf32"], "tf32x3": peaks["tf32"] / 3.0}[mode]
    tc_spec = {"bf16": SPEC["bf16"], "tf32": SPEC["tf32"], "tf32x3": SPEC["tf32"] / 3.0}[mode]
    gbs = kern_bytes / kern_s / 1e9
    tfs = kern_flops / kern_s / 1e12
    if kern_bytes / (peaks["hbm"] * 1e9) >= kern_flops / (tc_peak * 1e12):
        roof = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm"], "unit": "GB/s", "frac": gbs / peaks["hbm"],
                "spec_peak": SPEC["hbm"], "spec_frac": gbs / SPEC["hbm"]}
    else:
        roof = {"bound": "tensor", "achieved": tfs, "peak": tc_peak, "unit": "TFLOP/s", "frac": tfs / tc_peak,
                "spec_peak": tc_spec, "spec_frac": tfs / tc_spec}
    roof.update({"hbm_frac": gbs / peaks["hbm"], "tensor_frac": tfs / tc_peak,
                 "peak_source": peaks["source"] + ("; " + peaks["tf32_source"] if mode != "bf16" else ", bf16 burst")})
    return roof


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + clock-event reasons through NVML while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            log(f"[bench] NVML unavailable: {e}")
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for b, name in self.REASONS.items():
                    if bits & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self) -> dict:
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        self._stop.set()
        self._t.join()
        loaded = [s for s in self.samples]
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(loaded)}


# ----------------------------------------------------------------------------- inputs
def make_A_block(W, wl_name, r0, r1, c0, c1, device):
    """Rows [r0,r1) x cols [c0,c1) of the workload's A, generated in HBM (seeded)."""
    import torch
    from inputs import synth
    seed = SEED_A[wl_name]
    if W["a"] == "rbf":
        # RBF kernel block: rows r0..r1 of exp(-|x_i - x_j|^2 / 2 sigma^2), X ~ U[0,1)^{n x d}
        n, d = W["n1"], W["d"]
        g = torch.Generator(device=device)
        g.manual_seed(seed)
        X = torch.rand((n, d), generator=g, device=device, dtype=torch.float64)
        sigma2 = float((X * X).sum()) / n
        sq = (X * X).sum(1)
        out = torch.empty((r1 - r0, c1 - c0), dtype=torch.float32, device=device)
        step = 4096
        for i in range(r0, r1, step):
            ie = min(r1, i + step)
            d2 = (sq[i:ie, None] + sq[None, c0:c1] - 2.0 * (X[i:ie] @ X[c0:c1].T)).clamp_min_(0.0)
            out[i - r0:ie - r0] = torch.exp(-d2 / (2.0 * sigma2)).to(torch.float32)
        del X, sq
        torch.cuda.empty_cache()
        return out
    if W["a"] == "symuniform":
        A = torch.from_numpy(synth.symmetric_uniform(seed, W["n1"])).to(device)
        return A[r0:r1, c0:c1].contiguous()
    # iid U[-1/2, 1/2): generate row blocks with a per-(block) seed so any partition is reproducible
    out = torch.empty((r1 - r0, c1 - c0), dtype=torch.float32, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + r0 * 7 + c0)
    out.uniform_(-0.5, 0.5, generator=g)
    return out


def host_A_rows(W, wl_name, rows):
    """Host (numpy) copy of selected rows of A for the CPU oracle -- same recipe, host RNG."""
    import numpy as np
    from inputs import synth
    seed = SEED_A[wl_name]
    if W["a"] == "rbf":
        n, d = W["n1"], W["d"]
        X = np.random.Generator(np.random.PCG64(seed)).random((n, d))
        sigma2 = float((X * X).sum()) / n
        sq = (X * X).sum(1)
        d2 = np.maximum(sq[rows, None] + sq[None, :] - 2.0 * (X[rows] @ X.T), 0.0)
        return np.exp(-d2 / (2.0 * sigma2)).astype(np.float32)
    rng = np.random.Generator(np.random.PCG64(seed))
    return (rng.random((len(rows), W["n2"]), dtype=np.float32) - np.float32(0.5)).astype(np.float32)


# ----------------------------------------------------------------------------- oracle timing
def time_oracle(W, A_rows, target_s=12.0, cores=None):
    """Time the fp64 oracle (as it stands) on a bounded row sample; returns dict + B_sample."""
    import oracle
    if cores:
        oracle.set_num_threads(cores)
    n_rows = A_rows.shape[0]
    t0 = time.perf_counter()
    B = oracle.sketch(SEED_OMEGA, W["dist"], A_rows, W["r"])
    t = time.perf_counter() - t0
    return t, B


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, W, wl_name):
    import numpy as np
    import oracle
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count()
    oracle.set_num_threads(cores)
    # calibrate a row sample so that one step takes ~2-4 s of host time
    probe = 8
    A = host_A_rows(W, wl_name, list(range(probe)))
    t0 = time.perf_counter()
    oracle.sketch(SEED_OMEGA, W["dist"], A, W["r"])
    tp = time.perf_counter() - t0
    rows = int(max(8, min(W["n1"], probe * 3.0 / max(tp, 1e-3))))
    rows = min(rows, 4096)
    A = host_A_rows(W, wl_name, list(range(rows)))
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        B = oracle.sketch(SEED_OMEGA, W["dist"], A, W["r"])
        if W["nystrom"]:
            oracle.core(SEED_OMEGA, W["dist"], B, 0)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    gbs = rows * W["n2"] * 4 / t / 1e9
    sample = (f"{rows} of {W['n1']} rows of A per step (full K={W['n2']}, r={W['r']}); Omega "
              f"materialised in fp64 once per call" + ("; + Omega^T B of the sample rows" if W["nystrom"] else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": W["desc"], "n1": W["n1"], "n2": W["n2"], "r": W["r"], "dist": W["dist"],
                   "mode": "f64 oracle", "layout": "host", "sample_rows": rows},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ----------------------------------------------------------------------------- f4 ablation
def omega_ablation(args, W, sk, local, A, ds, dev, world, rank, stream, barrier, reps=5):
    """SURVEY §8f f4, the B200 version of Fig. 3 (regenerating Omega beats
    communicating it).  Same A block, B = A * Omega[K_j] only (no core), device time, max over ranks:
      fused        -- this library: Omega tiles regenerated inside the tcgen05 GEMM (never in HBM);
      materialise  -- Omega[K_j] generated into HBM by this library's generator kernel, then a cuBLAS
                      GEMM (torch.matmul; TF32 for tf32 modes; bf16 mode casts A and Omega first);
      allgather    -- (N > 1) each rank generates 1/N of Omega's rows, all_gather_into_tensor over
                      NCCL rebuilds Omega[K_j], then the same cuBLAS GEMM.
    cuBLAS is the comparison system here, not the product path."""
    import torch
    import torch.distributed as tdist
    r0, r1, c0, c1 = ds.a_block_range()
    k = c1 - c0
    r = local.r

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device=dev if world > 1 else "cpu")
        if world > 1:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t.item())

    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = args.mode != "tf32x3"
    out = {"omega_bytes_fp32": 4 * k * r, "a_block": [r1 - r0, k], "reps": reps,
           "gemm": "torch.matmul (cuBLAS), " + ("bf16 operands" if args.mode == "bf16" else
                                                  "TF32" if args.mode == "tf32" else "fp32")}
    Bbuf = torch.empty((r1 - r0, r), dtype=torch.float32, device=dev)
    out["fused_ms"] = timed(lambda: local.apply_block(A, c0, out=Bbuf))
    gen_ms = timed(lambda: local.generate(c0, k))
    Om = local.generate(c0, k)
    if args.mode == "bf16":
        gemm = lambda: torch.matmul(A.to(torch.bfloat16), Om.to(torch.bfloat16))
    else:
        gemm = lambda: torch.matmul(A, Om)
    out["materialise_generate_ms"] = gen_ms
    out["materialise_gemm_ms"] = timed(gemm)
    out["materialise_ms"] = gen_ms + out["materialise_gemm_ms"]
    if args.mode == "bf16":  # context: the fp32-operand (TF32) cuBLAS GEMM needs no cast of A
        torch.backends.cuda.matmul.allow_tf32 = True
        out["materialise_gemm_tf32_ms"] = timed(lambda: torch.matmul(A, Om))
    if world > 1:
        P = world
        per = -(-k // P)
        piece_rows = min(per, max(0, k - rank * per))
        piece = torch.zeros((per, r), dtype=torch.float32, device=dev)
        full = torch.empty((P * per, r), dtype=torch.float32, device=dev)

        def gather():
            if piece_rows:
                piece[:piece_rows].copy_(local.generate(c0 + rank * per, piece_rows))
            tdist.all_gather_into_tensor(full, piece)

        out["allgather_generate_and_gather_ms"] = timed(gather)
        out["allgather_ms"] = out["allgather_generate_and_gather_ms"] + out["materialise_gemm_ms"]
    torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    del Om
    return out


# ----------------------------------------------------------------------------- our arm
def relaunch_under_torchrun(n: int) -> None:
    """Re-executes this command as `torch.distributed.run --nproc-per-node n` on 127.0.0.1 and exits
    with its status (rank 0 prints the JSON line)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("[bench] launching " + " ".join(cmd[1:]))
    sys.exit(subprocess.call(cmd, stdout=_JSON_FD if _JSON_FD is not None else None))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="bf16", choices=["tf32", "tf32x3", "bf16"])
    ap.add_argument("--omega", default="auto", choices=["auto", "accurate", "fast"],
                    help="Gaussian transform: auto = fast (MUFU Box-Muller, error <= 2^-18 max(|z|,1), measured 2^-18.96) in bf16 "
                         "mode, whose RN rounding of Omega to bf16 (2^-9) hides it (same relF of B as accurate), "
                         "accurate (<= 2 ulp fp32) in tf32 / tf32x3 (reading R5)")
    ap.add_argument("--layout", default="auto",
                    help="row | col | AxB (p1 x p2) | auto = the grid BASELINE.json names: c2 / c5 the most "
                         "square 2D grid, c3 row-block, c4 column-block")
    ap.add_argument("--split-k", type=int, default=0)
    ap.add_argument("--variant", default="noredist", choices=["noredist", "redist"],
                    help="Alg. 2 variant for N > 1 row-block Nystrom (PAPER.md:698)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the timed steps as CUDA graphs (auto = on); the per-phase kernel times then come "
                         "from the profiled eager pass that precedes them")
    ap.add_argument("--nccl-ar", action="store_true",
                    help="AllReduce C with NCCL instead of the default fused NVLink peer-read sum (f1, symmetric memory)")
    ap.add_argument("--ar", default="sum", choices=["sum", "epilogue"],
                    help="AllReduce of C over symmetric memory: a fixed-order sum after one barrier (default), "
                         "or issued from the core GEMM's epilogue as in-switch multimem reductions (f1)")
    ap.add_argument("--rs", default="peer", choices=["nccl", "peer", "epilogue"],
                    help="reduce-scatter of partial B in column / 2D layouts: NCCL, symmetric-memory peer-read "
                         "sum (default), or stores from the GEMM epilogue into the owners' slots (f1)")
    ap.add_argument("--omega-ablation", action="store_true",
                    help="f4: also time B = A*Omega with Omega materialised in HBM (+ all-gathered over NCCL "
                         "when N > 1) and a cuBLAS GEMM, against the fused in-kernel regeneration")
    ap.add_argument("--balance", action="store_true",
                    help="row-block grids: whole cluster units per rank with the ragged tail rows split by columns "
                         "and reduced onto the last rank (measured no faster at 2 / 4 GPUs: the tail launch's "
                         "unshared Omega costs what the saved unit saves), instead of the plain balanced row split")
    ap.add_argument("--no-other-modes", action="store_true",
                    help="skip timing the other precision modes / transforms after the main line")
    args = ap.parse_args()
    W = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, W, args.workload)
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        # `bench.py --gpus N` outside a launcher: start the N ranks (one process per GPU) ourselves
        return relaunch_under_torchrun(args.gpus)
    if ws_env is not None and int(ws_env) != args.gpus:
        log(f"[bench] --gpus {args.gpus} does not match WORLD_SIZE={ws_env}; refusing to run")
        sys.exit(2)
    args.warmup = max(args.warmup, 3)
    if args.omega == "auto":
        args.omega = "fast" if args.mode == "bf16" else "accurate"

    import numpy as np
    import torch
    import torch.distributed as tdist

    import paper_2603_20966_b200 as sk
    from paper_2603_20966_b200.dist import DistSketch, Layout, predicted_bytes_per_rank

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        tdist.init_process_group("nccl", device_id=dev)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        tdist.init_process_group("gloo", rank=0, world_size=1)
    layout = Layout.parse(auto_layout(args.workload, world) if args.layout == "auto" else args.layout, world)
    n1, n2, r = W["n1"], W["n2"], W["r"]
    peaks = load_peaks()

    local = sk.Sketch(SEED_OMEGA, W["dist"], n2, r, mode=args.mode, omega=args.omega, split_k=args.split_k)
    # row-block grids cut at whole units of the library's plan (the ragged tail split by columns)
    unit = 0
    if layout.p2 == 1 and world > 1 and args.balance:
        unit = local.plan_info(-(-n1 // world), n2)["rows_per_unit"]
    ds = DistSketch(SEED_OMEGA, W["dist"], n1, n2, r, layout, local=local, fused_rs=args.rs,
                    fused_ar=("epilogue" if args.ar == "epilogue" else not args.nccl_ar), balance_unit=unit)
    r0, r1, c0, c1 = ds.a_block_range()
    t_gen = time.perf_counter()
    A = make_A_block(W, args.workload, r0, r1, c0, c1, dev)
    tail = ds.tail_block_range()
    A_tail = make_A_block(W, args.workload, *tail, dev) if tail is not None else None
    torch.cuda.synchronize()
    log(f"[bench] rank {rank}: A block {tuple(A.shape)}" + (f" + tail block {tuple(A_tail.shape)}" if tail else "") +
        f" generated in {time.perf_counter() - t_gen:.1f}s")
    stream = torch.cuda.current_stream()

    def step():
        if W["nystrom"] and args.variant == "redist" and world > 1:
            return ds.nystrom_core_redist(A, A_tail)
        if W["nystrom"]:
            return ds.nystrom_core(A, A_tail)
        Bp, rows = ds.apply(A, A_tail)
        return Bp, rows, None

    def barrier():
        if world > 1:
            tdist.barrier(device_ids=[local_rank])

    for _ in range(args.warmup):
        out = step()
    torch.cuda.synchronize()
    barrier()

    # ------------------------------------------------------------------ timed region
    sampler = ClockSampler(local_rank)
    local.set_profiling(True)
    local.profile_read()  # clear
    launches0 = sk.launch_count()
    ds.comm_bytes = 0
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e0.record(stream)
    h0 = time.perf_counter()
    for i in range(args.steps):
        out = step()
        step_ev[i].record(stream)  # per-step boundaries (median); the total is e0 -> e1
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # host submission time per step
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    per_step = [e0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i]) for i in range(1, args.steps)]
    launches = sk.launch_count() - launches0
    comm_bytes = ds.comm_bytes / args.steps  # python-side accounting of the eager timed steps
    phases = local.profile_read()
    local.set_profiling(False)
    t_ms = e0.elapsed_time(e1)
    use_graph = args.graph == "on" or args.graph == "auto"
    graph_info = None
    eager_ms_step = t_ms / args.steps
    if use_graph and world > 1:
        # N > 1: the step (sketch, split-K reduce, symmetric-memory barriers, reduce-scatter / AllReduce
        # kernels, core GEMM) captured as CUDA graphs and replayed; two steps per graph so the
        # alternating receive slots keep alternating (plus a one-step graph for an odd K).  All ranks
        # capture in lockstep and agree on success before replaying.
        gerr = None
        try:
            gs = torch.cuda.Stream()
            gs.wait_stream(stream)
            with torch.cuda.stream(gs):
                for _ in range(2):
                    out = step()
            stream.wait_stream(gs)
            torch.cuda.synchronize()
            g2 = torch.cuda.CUDAGraph()
            lc0 = sk.launch_count()
            with torch.cuda.graph(g2, stream=gs):
                step()
                out = step()
            launches_per_step = (sk.launch_count() - lc0) / 2.0
            g1 = None
            if args.steps % 2:
                g1 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g1, stream=gs):
                    out = step()
        except Exception as e:  # pragma: no cover - capture unsupported here
            gerr = repr(e)
        okt = torch.tensor([0 if gerr else 1], dtype=torch.int32, device=dev)
        tdist.all_reduce(okt, op=tdist.ReduceOp.MIN)
        if int(okt.item()) == 1:
            for _ in range(max(2, args.warmup // 2)):
                g2.replay()
            torch.cuda.synchronize()
            barrier()
            torch.cuda.synchronize()
            npair = args.steps // 2
            pair_ev = [torch.cuda.Event(enable_timing=True) for _ in range(max(npair, 1))]
            e0.record(stream)
            h0 = time.perf_counter()
            for i in range(npair):
                g2.replay()
                pair_ev[i].record(stream)
            if g1 is not None:
                g1.replay()
            host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            t_ms = e0.elapsed_time(e1)
            if npair:
                per_step = [e0.elapsed_time(pair_ev[0]) / 2.0] + [pair_ev[i - 1].elapsed_time(pair_ev[i]) / 2.0
                                                                  for i in range(1, npair)]
            launches = int(round(launches_per_step * args.steps))
            graph_info = {"replayed": True, "steps_per_graph": 2, "launches_per_step": launches_per_step,
                          "eager_ms_per_step": eager_ms_step}
        else:
            graph_info = {"replayed": False, "error": gerr or "capture failed on another rank"}
    if use_graph and world == 1:
        # the step captured once as a CUDA graph (library launches on the capture stream) and replayed:
        # the eager pass above supplied the per-phase kernel times
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        with torch.cuda.stream(gs):
            for _ in range(2):
                out = step()
        stream.wait_stream(gs)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        lc0 = sk.launch_count()
        with torch.cuda.graph(g, stream=gs):
            out = step()
        launches_per_step = sk.launch_count() - lc0
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        e0.record(stream)
        h0 = time.perf_counter()
        for i in range(args.steps):
            g.replay()
            step_ev[i].record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        e1.record(stream)
        torch.cuda.synchronize()
        t_ms = e0.elapsed_time(e1)
        per_step = [e0.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i])
                                                    for i in range(1, args.steps)]
        launches = launches_per_step * args.steps
        graph_info = {"replayed": True, "launches_per_step": launches_per_step,
                      "eager_ms_per_step": eager_ms_step}
    clocks = sampler.stop()
    tmax = torch.tensor([t_ms], dtype=torch.float64, device=dev if world > 1 else "cpu")
    if world > 1:
        tdist.all_reduce(tmax, op=tdist.ReduceOp.MAX)
    t_ms = float(tmax.item())
    ms_step = t_ms / args.steps
    med = torch.tensor([statistics.median(per_step)], dtype=torch.float64, device=dev if world > 1 else "cpu")
    if world > 1:
        tdist.all_reduce(med, op=tdist.ReduceOp.MAX)
    ms_step_median = float(med.item())
    a_bytes_total = 4.0 * n1 * n2
    value = a_bytes_total / (ms_step * 1e-3) / 1e9
    flops = 2.0 * n1 * n2 * r + (2.0 * n2 * r * r if W["nystrom"] else 0.0)
    tflops = flops / (ms_step * 1e-3) / 1e12

    # ------------------------------------------------------------------ roofline (dominant kernel)
    gemm_ms, gemm_launches = phases["sketch_gemm"]
    m_loc, k_loc = (r1 - r0), (c1 - c0)
    kern_bytes = 4.0 * m_loc * k_loc + 4.0 * m_loc * r  # A read + B write (algorithmic)
    kern_flops = 2.0 * m_loc * k_loc * r
    avg_s = (gemm_ms / max(gemm_launches, 1)) * 1e-3
    passes = max(1, gemm_launches // max(args.steps, 1))
    avg_s_step = avg_s * passes  # all column passes of one step
    roof = roofline(args.mode, kern_bytes, kern_flops, avg_s_step, peaks)
    roof.update({
        "kernel": f"sketch_gemm_kernel (fused Philox/Box-Muller Omega tiles + tcgen05 {args.mode})",
        "launches_timed": gemm_launches, "avg_launch_ms": avg_s * 1e3,
        "share_of_step": (gemm_ms / max(t_ms, 1e-9)),
        "traffic": None,
    })
    prof_path = os.path.join(ROOT, "profiles", f"traffic_{args.workload}_{args.mode}_{args.omega}.json")
    if os.path.exists(prof_path) and world == 1:  # the capture is of the 1-GPU launch
        with open(prof_path) as f:
            tr = json.load(f)
        roof["traffic"] = tr.get("dram_bytes_per_launch")
        roof["traffic_source"] = os.path.relpath(prof_path, ROOT)

    result = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "ms_per_step_median": ms_step_median,
        "value_median": a_bytes_total / (ms_step_median * 1e-3) / 1e9, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.mode, "data": "synthetic (seeded, generated in HBM)",
        "config": {"workload": W["desc"], "n1": n1, "n2": n2, "r": r, "dist": W["dist"], "mode": args.mode,
                   "omega_transform": args.omega, "layout": f"{layout.p1}x{layout.p2}",
                   "row_split": (f"{ds.tail['M']} rows per rank (whole units of {unit}) + the {ds.tail['R']}-row tail "
                                 f"split by columns, reduced onto rank {world - 1}" if ds.tail else "balanced"),
                   "layout_rule": ("BASELINE.json's 2D grid (most square p1 x p2, p1 >= p2)"
                                   if args.layout == "auto" and W["nystrom"] else args.layout),
                   "l2": "inputs larger than L2 (A = %.1f GB)" % (a_bytes_total / 1e9) if a_bytes_total > 126e6
                   else "A fits in L2 (c1: launch-latency bound)"},
        "tflops": tflops,
        "nystrom_core_ms": ms_step if W["nystrom"] else None,
        "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items() if v[1]},
        "roofline": roof,
        "gpu_launches": launches,
        "host_submit_ms_per_step": host_ms,
        "cuda_graph": graph_info,
        "clocks": clocks,
        "comm": {"variant": args.variant if (W["nystrom"] and world > 1) else None,
                 "reduce_scatter": ds.rs_mode,
                 "fused_allreduce": bool(ds.fused_ar and world > 1),
                 "symmetric_reduce_path": ds.reduce_path,  # "nvls" (in-switch multimem) / "peer" (NVLink reads)
                 "predicted_bytes_per_rank": predicted_bytes_per_rank(n1, r, layout, W["nystrom"],
                                                                     args.variant if world > 1 else "noredist",
                                                                     tail_rows=ds.tail["R"] if ds.tail else 0),
                 "measured_bytes_per_rank": comm_bytes},
    }

    # ------------------------------------------------------------------ the other modes (same A, same step)
    if not args.no_other_modes:
        others = {}
        for mode, omega in (("tf32x3", "accurate"), ("tf32", "accurate"), ("tf32", "fast"), ("bf16", "accurate"),
                            ("bf16", "fast")):
            if (mode, omega) == (args.mode, args.omega):
                continue
            try:
                loc2 = sk.Sketch(SEED_OMEGA, W["dist"], n2, r, mode=mode, omega=omega)
                ds2 = DistSketch(SEED_OMEGA, W["dist"], n1, n2, r, layout, local=loc2)

                def step2():
                    return ds2.nystrom_core(A) if W["nystrom"] else ds2.apply(A)

                for _ in range(3):
                    step2()
                torch.cuda.synchronize()
                barrier()
                reps = max(3, args.steps // 2)
                loc2.set_profiling(True)
                loc2.profile_read()
                g0 = torch.cuda.Event(enable_timing=True)
                g1 = torch.cuda.Event(enable_timing=True)
                g0.record(stream)
                for _ in range(reps):
                    step2()
                g1.record(stream)
                torch.cuda.synchronize()
                ph2 = loc2.profile_read()
                loc2.set_profiling(False)
                t2 = torch.tensor([g0.elapsed_time(g1) / reps], dtype=torch.float64,
                                  device=dev if world > 1 else "cpu")
                if world > 1:
                    tdist.all_reduce(t2, op=tdist.ReduceOp.MAX)
                t2 = float(t2.item())
                sk_s = ph2["sketch_gemm"][0] / reps * 1e-3  # sketch kernel time per step (all its launches)
                others[f"{mode}/{omega}"] = {
                    "ms_per_step": t2, "value": a_bytes_total / (t2 * 1e-3) / 1e9,
                    "phases_ms_per_step": {k: v[0] / reps for k, v in ph2.items() if v[1]},
                    "roofline": roofline(mode, kern_bytes, kern_flops, sk_s, peaks) if sk_s > 0 else None}
                del loc2, ds2
            except Exception as e:  # pragma: no cover
                others[f"{mode}/{omega}"] = {"error": repr(e)}
        result["other_modes"] = others

    # ------------------------------------------------------------------ f4: regenerate vs materialise / gather
    if args.omega_ablation:
        result["omega_ablation"] = omega_ablation(args, W, sk, local, A, ds, dev, world, rank, stream, barrier)

    # ------------------------------------------------------------------ parity at full size (sampled)
    if rank == 0 and not args.no_parity:
        try:
            import oracle
            Bp, (a, b), C = out
            rows = sorted(set(int(x) for x in np.linspace(a, min(b, a + A.shape[0]) - 1, 24)))  # bulk block rows
            # the exact device rows of A (and, for row-block layouts, all of K) go to the oracle
            A_rows = A[[x - r0 for x in rows]].cpu().numpy() if (c0, c1) == (0, n2) else None
            if A_rows is not None:
                Bref = oracle.sketch(SEED_OMEGA, W["dist"], A_rows, r)
                Bg = Bp[[x - a for x in rows]].double().cpu().numpy()
                relB = float(np.linalg.norm(Bg - Bref) / np.linalg.norm(Bref))
                par = {"rows_sampled": len(rows), "relF_B_rows": relB}
                if W["nystrom"] and world == 1:
                    Cown = oracle.core(SEED_OMEGA, W["dist"], Bp.double().cpu().numpy(), 0)
                    Cg = C.double().cpu().numpy()
                    par["relF_C_vs_oracle_core_of_gpu_B"] = float(np.linalg.norm(Cg - Cown) / np.linalg.norm(Cown))
                    par["C_symmetry_relF"] = float(np.linalg.norm(Cg - Cg.T) / np.linalg.norm(Cg))
                result["parity"] = par
        except Exception as e:  # pragma: no cover
            result["parity"] = {"error": repr(e)}

    # ------------------------------------------------------------------ cpu baseline (oracle)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            cores = os.cpu_count()
            oracle.set_num_threads(cores)
            # grow the row sample until the oracle runs >= ~10 s (it materialises Omega once per call,
            # a fixed cost, so a small probe would under-size the sample)
            nrows, t = 32, 0.0
            while True:
                A_rows = A[:nrows].cpu().numpy()
                t, _ = time_oracle(W, A_rows)
                if t >= 10.0 or nrows >= min(A.shape[0], 16384):
                    break
                nrows = int(min(min(A.shape[0], 16384), max(2 * nrows, nrows * 12.0 / max(t, 1e-3))))
            # the paper's phase split (genOmegaTime / dgemm1Time): the oracle's
            # materialisation of Omega alone, the rest of the call is the fp64 GEMM
            t0 = time.perf_counter()
            oracle.omega(SEED_OMEGA, W["dist"], 0, n2, 0, r)
            t_om = time.perf_counter() - t0
            result["cpu_baseline"] = {
                "value": nrows * n2 * 4 / t / 1e9, "unit": "GB/s", "cores": oracle.num_threads(),
                "kind": "oracle",
                "sample": f"B = A Omega for rows 0..{nrows - 1} of {n1} (full K={n2}, r={r}), fp64, "
                          f"Omega materialised once; {t:.1f} s",
                "phases_s": {"gen_omega": t_om, "gemm": max(t - t_om, 0.0)},
            }
        except Exception as e:  # pragma: no cover
            result["cpu_baseline"] = {"error": repr(e)}

    # ------------------------------------------------------------------ e2e (host buffers, through the ABI)
    # The same step through the host-buffer entry points (sketch_apply_host / nystrom_core_host):
    # this rank's A block starts in pinned host memory; the library streams it in row blocks
    # (H2D of block i+1 overlapped with the sketch of block i), copies B back, and accumulates C;
    # for N > 1 the r x r C partials are then all-reduced as in the device path.
    if not args.no_e2e:
        try:
            Ah = torch.empty(A.shape, dtype=torch.float32, pin_memory=True)
            Ah.copy_(A)
            pa, pb = ds.b_piece_rows()
            rows_b = pb - pa
            Bh = torch.empty((rows_b, r), dtype=torch.float32, pin_memory=True)
            Ch = torch.empty((r, r), dtype=torch.float32, pin_memory=True)
            host_row_layout = (c0, c1) == (0, n2) and tail is None
            Aht = None
            if tail is not None:
                Aht = torch.empty(A_tail.shape, dtype=torch.float32, pin_memory=True)
                Aht.copy_(A_tail)

            def e2e_step():
                if W["nystrom"] and host_row_layout:
                    if world == 1:
                        local.nystrom_core_host(Ah, B=Bh, C=Ch, sync=False)
                    else:
                        local.apply_host(Ah, out=Bh, sync=False)
                        Bd = Bh.to(dev, non_blocking=True)
                        Cd = local.core_block(Bd, r0)
                        tdist.all_reduce(Cd)
                        Ch.copy_(Cd, non_blocking=True)
                elif host_row_layout:
                    local.apply_host(Ah, out=Bh, sync=False)
                else:  # column / 2D / balanced layouts: stage this rank's block(s), then the device path
                    A.copy_(Ah, non_blocking=True)
                    if Aht is not None:
                        A_tail.copy_(Aht, non_blocking=True)
                    o = step()
                    Bh[: o[0].shape[0]].copy_(o[0], non_blocking=True)
                    if o[2] is not None:
                        Ch.copy_(o[2], non_blocking=True)

            e2e_step()  # warm-up (workspace allocation)
            torch.cuda.synchronize()
            barrier()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(args.e2e_steps):
                e2e_step()
            f1.record(stream)
            torch.cuda.synchronize()
            te = torch.tensor([f0.elapsed_time(f1) / args.e2e_steps], dtype=torch.float64,
                              device=dev if world > 1 else "cpu")
            if world > 1:
                tdist.all_reduce(te, op=tdist.ReduceOp.MAX)
            te = float(te.item())
            result["e2e"] = {"value": a_bytes_total / (te * 1e-3) / 1e9, "unit": "GB/s",
                             "h2d_bytes_per_step": int(A.numel() * 4 + (A_tail.numel() * 4 if A_tail is not None else 0)),
                             "d2h_bytes_per_step": int(Bh.numel() * 4 + (Ch.numel() * 4 if W["nystrom"] else 0)),
                             "ms_per_step": te,
                             "path": ("nystrom_core_host / sketch_apply_host (C ABI, pinned host A streamed in row "
                                      "blocks, H2D overlapped with compute, B and C copied back)" if host_row_layout
                                      else "pinned host A block -> H2D, then the device path, D2H of B and C")}
            del Ah
        except Exception as e:  # pragma: no cover
            result["e2e"] = {"error": repr(e)}

    if rank == 0:
        emit(result)
    if world > 1:
        tdist.barrier(device_ids=[local_rank])
    tdist.destroy_process_group()


if __name__ == "__main__":
    _stdout_to_stderr()
    main()
