"""The device Philox4x32-10 of the library against NVIDIA cuRAND's own implementation
(curand_Philox4x32_10, compiled from curand_kernel.h into a test-only .so), bit for bit, through the
library's Omega-word entry point sketch_generate_bits -- an independent pin of the on-GPU generator in
addition to the Random123 known-answer vectors.  Also: the in-GEMM Omega is
prefix-consistent in r (the first 128 columns of an r = 256 sketch equal the r = 128 sketch, bit for
bit, in the integer regime)."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 0x1234_5678_9ABC_DEF0


def _curand_lib(tmp_path_factory):
    src = os.path.join(HERE, "cuda", "curand_ref.cu")
    out = str(tmp_path_factory.mktemp("curand") / "libcurand_ref.so")
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-shared",
                    "-Xcompiler", "-fPIC", src, "-o", out], check=True)
    lib = ctypes.CDLL(out)
    lib.curand_philox_words.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("dist,tag", [("gaussian", 0), ("rademacher", 1)])
def test_library_philox_matches_curand(dist, tag, tmp_path_factory):
    import paper_2603_20966_b200 as sk
    lib = _curand_lib(tmp_path_factory)
    n2, r = 1 << 20, 96
    s = sk.Sketch(SEED, dist, n2, r)
    rows = np.array([0, 1, 2, 3, 4, 127, 128, 129, 12345, 1000003, n2 - 1], dtype=np.int64)
    cols = np.array([0, 1, 31, 32, 95], dtype=np.int64)
    words = {}
    for j in rows:
        w = s.generate_bits(int(j), 1).cpu().numpy().view(np.uint32)[0]
        for k in cols:
            words[(int(j), int(k))] = int(w[k])
    # the same entries from cuRAND: counter (q lo, q hi, k, tag), q = j >> 2 (tag 0) / j >> 7 (tag 1)
    keys = list(words)
    ctr = np.zeros((len(keys), 4), dtype=np.uint32)
    key = np.zeros((len(keys), 2), dtype=np.uint32)
    for i, (j, k) in enumerate(keys):
        q = j >> 2 if tag == 0 else j >> 7
        ctr[i] = (q & 0xFFFFFFFF, q >> 32, k, tag)
        key[i] = (SEED & 0xFFFFFFFF, SEED >> 32)
    dc, dk = torch.from_numpy(ctr.view(np.int32)).cuda(), torch.from_numpy(key.view(np.int32)).cuda()
    out = torch.empty((len(keys), 4), dtype=torch.int32, device="cuda")
    assert lib.curand_philox_words(dc.data_ptr(), dk.data_ptr(), len(keys), out.data_ptr()) == 0
    ref = out.cpu().numpy().view(np.uint32)
    for i, (j, k) in enumerate(keys):
        # generate_bits returns, per O1, word j & 3 of the call (tag 0) / word (j >> 5) & 3 (tag 1)
        sel = j & 3 if tag == 0 else (j >> 5) & 3
        assert words[(j, k)] == int(ref[i, sel]), (j, k)


def test_in_gemm_omega_prefix_consistent_in_r():
    import paper_2603_20966_b200 as sk
    from inputs import synth
    A = torch.from_numpy(synth.int_matrix(61, 900, 2500)).cuda()
    for mode in ("tf32", "bf16"):
        B256 = sk.Sketch(42, "rademacher", 2500, 256, mode=mode).apply(A)
        B128 = sk.Sketch(42, "rademacher", 2500, 128, mode=mode).apply(A)
        assert torch.equal(B256[:, :128], B128), mode
