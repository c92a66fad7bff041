"""K3f: the last level's output step C_k = sum_r w_kr M_r fused into the
leaf GEMM's epilogue (option fuse_output): every leaf tile is reduce-added by TMA into the output
sub-blocks its W column touches.  The order of those fp64 adds is not fixed, so parity is checked
bit-exactly on integer inputs (every partial sum is an exact integer) and by tolerance on uniform
inputs, against the oracle."""
import os

import numpy as np
import pytest

import fmm_inputs as I
from conftest import ALGS
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _F():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


def _dev(x, layout):
    if layout == "row":
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()


@pytest.mark.parametrize("alg,L,shape,layout", [
    ("strassen_222_7", 1, (256, 256, 256), "row"),
    ("winograd_class_222_7", 2, (520, 264, 392), "col"),
    ("hk_class_323_15", 2, (302, 200, 262), "row"),        # peeled at both levels
    ("alg_424_26", 2, (1000, 300, 1000), "row"),           # ragged leaf tiles: zero rows spill into neighbours
    ("alg_433_29", 2, (1128, 360, 400), "col"),
    ("laderman_class_333_23", 1, (300, 300, 300), "row"),
    ("flip_234_20", 2, (200, 336, 400), "row")])
def test_k3f_integer_exact(alg, L, shape, layout):
    F = _F()
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=51, kind="integers")
    p = F.Plan(F.load_alg(alg), P, Q, N, L, layout=layout, fuse_output=True)
    assert p.stats()["fused_output"] == 1
    want = A @ B
    for _ in range(3):  # plain launches, then CUDA-graph capture and replay
        C = p.execute(_dev(A, layout), _dev(B, layout))
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), want)


@pytest.mark.parametrize("alg,L,shape", [("alg_424_26", 2, (2000, 600, 2000)), ("winograd_class_222_7", 2, (1024, 1024, 1024))])
def test_k3f_uniform_within_tolerance(alg, L, shape):
    F = _F()
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=52)
    p = F.Plan(F.load_alg(alg), P, Q, N, L, fuse_output=True)
    C = p.execute(_dev(A, "row"), _dev(B, "row")).cpu().numpy()
    ref = O.fast(A, B, O.load_alg(os.path.join(ALGS, alg + ".txt")), L)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(C - ref)) <= 1e-12 * nrm
    assert np.max(np.abs(C - O.classical(A, B))) <= 1e-10 * nrm


def test_k3f_not_applied_where_it_cannot_be():
    # a rational W coefficient (not +-1): the plan keeps the separate assembly
    F = _F()
    from fractions import Fraction as Fr
    s = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    U = [[v * (2 if r == 0 else 1) for r, v in enumerate(row)] for row in s.U]
    W = [[v * (Fr(1, 2) if r == 0 else 1) for r, v in enumerate(row)] for row in s.W]
    a = F.Algorithm.create(2, 2, 2, 7, U, s.V, W)
    p = F.Plan(a, 64, 64, 64, 1, fuse_output=True)
    assert p.stats()["fused_output"] == 0
    A, B = I.problem(64, 64, 64, seed=53, kind="integers")
    assert np.array_equal(p.execute(_dev(A, "row"), _dev(B, "row")).cpu().numpy(), A @ B)


def test_k3f_needs_tma_views():
    # an odd leading dimension cannot be described to TMA: the execute says so before any device work
    F = _F()
    A, B = I.problem(301, 199, 257, seed=54, kind="integers")
    p = F.Plan(F.load_alg("hk_class_323_15"), 301, 199, 257, 2, fuse_output=True)
    with pytest.raises(F.FmmError) as e:
        p.execute(_dev(A, "row"), _dev(B, "row"))
    assert e.value.status == "FMM_E_UNSUPPORTED"
