"""bench.py contract on the GPU (small workload): one JSON line with the required keys, and the f4
Omega ablation (fused regeneration vs materialised Omega + cuBLAS) agreeing on what it times."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_c1_line_and_omega_ablation():
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", "c1", "--mode", "tf32", "--steps", "3",
           "--warmup", "3", "--no-other-modes", "--no-cpu-baseline", "--omega-ablation"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in line, key
    assert line["gpu_launches"] > 0
    ab = line["omega_ablation"]
    assert ab["omega_bytes_fp32"] == 4 * 512 * 16
    for key in ("fused_ms", "materialise_generate_ms", "materialise_gemm_ms", "materialise_ms"):
        assert ab[key] > 0
