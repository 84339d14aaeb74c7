"""Seeded random sweep of the multi-GPU paths on ONE GPU through virtual ranks (tests/test_virtual_gpu.py):
random sizes (ragged blocks included), rank counts, grids, reduce-scatter kinds, Nystrom variants and
modes, all in the integer regime, so every rank's B piece and the replicated C must equal the fp64
oracle of the whole problem bit for bit.  Alg. 1, Alg. 2 No-Redist
 and Redist.
"""
import numpy as np
import pytest

import oracle
from inputs import synth
from tests.test_virtual_gpu import SEED, _check_exact, _run

pytestmark = pytest.mark.gpu

GRIDS = {2: ["row", "col"], 4: ["row", "col", "2x2"], 8: ["row", "col", "4x2", "2x4"]}
NCASES = 96


def _case(i):
    g = np.random.default_rng(2000 + i)
    world = int(g.choice([2, 4, 8]))
    spec = str(g.choice(GRIDS[world]))
    square = g.random() < 0.6
    n1 = int(g.integers(world * 16, 3000))
    n2 = n1 if square else int(g.integers(world * 16, 6000))
    r = int(g.choice([8, 24, 40, 64, 100, 128]))
    mode = str(g.choice(["tf32x3", "tf32", "bf16"]))
    p2 = 1 if spec == "row" else world if spec == "col" else int(spec.split("x")[1])
    rs = "nccl" if p2 == 1 else str(g.choice(["nccl", "peer", "epilogue"]))
    variant = "redist" if square and spec == "row" and g.random() < 0.5 else "noredist"
    # Redist: the r columns of C split as evenly as they allow (r = 100 over 8 ranks: 13 / 12 columns)
    return dict(world=world, spec=spec, n1=n1, n2=n2, r=r, mode=mode, rs=rs, variant=variant)


@pytest.mark.parametrize("i", range(NCASES))
def test_virtual_fuzz_case(i):
    c = _case(i)
    square = c["n1"] == c["n2"]
    A = synth.int_matrix(100 + i, c["n1"], c["n2"], -4, 4, symmetric=square)
    if square:
        Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, c["r"])
    else:
        Bref, Cref = oracle.sketch(SEED, "rademacher", A, c["r"]), None
    res = _run(c["world"], c["spec"], c["n1"], c["n2"], c["r"], "rademacher", c["mode"], A, rs=c["rs"],
               fused_ar=square, variant=c["variant"])
    _check_exact(res, Bref, Cref, c["n1"])
    for rk in res:
        assert not rk["fallbacks"], (c, rk["fallbacks"])


@pytest.mark.parametrize("world,r,mode", [(8, 100, "bf16"), (4, 30, "tf32x3"), (2, 7, "tf32")])
def test_virtual_redist_ragged_columns(world, r, mode):
    """Redist with r not a multiple of P: the column blocks of C differ by one column."""
    n = 1333
    A = synth.int_matrix(17, n, n, -4, 4, symmetric=True)
    Bref, Cref = oracle.nystrom_core(SEED, "rademacher", A, r)
    res = _run(world, "row", n, n, r, "rademacher", mode, A, variant="redist")
    _check_exact(res, Bref, Cref, n)
