"""Collapsed levels (collapse_levels = 1): the formation and assembly of the last
two recursion levels in one streaming pass each; the level-(L-1) S_r, T_r, M_r are never written.

The two-level chains are the oracle's two levels in the oracle's order, so with CSE off the
collapsed and the one-level-per-launch schedules agree bitwise; both meet the north-star tolerance
against the oracle; integer inputs are exact; leaf shards still sum to the product; a plan that
cannot collapse (peeling at level L-1, a large base case, write-once) silently uses the separate
kernels.
"""
import numpy as np
import pytest

import fmm_inputs as I
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


def _run(F, name, A, B, L, layout="row", **kw):
    import torch
    P, Q = A.shape
    N = B.shape[1]

    def dev(x):
        if layout == "row":
            return torch.from_numpy(np.ascontiguousarray(x)).cuda()
        return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    p = F.Plan(F.load_alg(name), P, Q, N, L, layout=layout, **kw)
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy(), p.stats()


CASES = [("strassen_222_7", 256, 256, 256, 2, "row"), ("winograd_class_222_7", 1024, 1024, 1024, 2, "col"),
         ("winograd_class_222_7", 2048, 512, 1536, 2, "row"), ("strassen_222_7", 1000, 992, 1008, 2, "row"),  # odd-width leaves
         ("strassen_222_7", 1024, 512, 768, 3, "col"), ("winograd_class_222_7", 64, 64, 64, 2, "row")]


@pytest.mark.parametrize("name,P,Q,N,L,layout", CASES)
def test_collapsed_equals_separate_and_oracle(name, P, Q, N, L, layout):
    F = _lib()
    A, B = I.problem(P, Q, N, seed=P + L)
    Cc, sc = _run(F, name, A, B, L, layout, cse=False, collapse=True)
    Cs, ss = _run(F, name, A, B, L, layout, cse=False, collapse=False)
    assert sc["add_bytes"] < ss["add_bytes"] and sc["launches"] < ss["launches"]  # it did collapse
    assert np.array_equal(Cc, Cs)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(Cc - O.fast(A, B, O.load_alg(F.alg_path(name)), L))) <= 1e-12 * nrm
    assert np.max(np.abs(Cc - O.classical(A, B))) <= 1e-10 * nrm


@pytest.mark.parametrize("name", ["strassen_222_7", "winograd_class_222_7"])
def test_collapsed_integer_exact(name):
    F = _lib()
    A, B = I.problem(384, 256, 320, seed=3, kind="integers")
    C, st = _run(F, name, A, B, 2)
    assert np.array_equal(C, A @ B)


@pytest.mark.parametrize("G", [2, 3, 8])
def test_collapsed_shards_sum_to_product(G):
    F = _lib()
    A, B = I.problem(256, 192, 320, seed=8, kind="integers")
    total = np.zeros((256, 320))
    for g in range(G):
        C, _ = _run(F, "winograd_class_222_7", A, B, 2, shard_rank=g, shard_count=G)
        total += C
    assert np.array_equal(total, A @ B)


def test_not_collapsed_where_it_does_not_apply():
    F = _lib()
    A, B = I.problem(250, 250, 250, seed=4, kind="integers")  # 250 -> 125: peeled at level 1 = L-1
    Ca, sa = _run(F, "strassen_222_7", A, B, 2, collapse=True)
    Cb, sb = _run(F, "strassen_222_7", A, B, 2, collapse=False)
    assert sa["launches"] == sb["launches"] and np.array_equal(Ca, A @ B) and np.array_equal(Cb, A @ B)
    A, B = I.problem(540, 360, 540, seed=5, kind="integers")  # <3,2,3>: base case too large (the wide
    Ca, sa = _run(F, "hk_class_323_15", A, B, 2, collapse=True)  # assembly and the formation alone only on
    _, sb = _run(F, "hk_class_323_15", A, B, 2, collapse=False)  # request)
    assert sa["collapsed"] == 0 and sa["collapsed_assembly"] == 0 and sa["launches"] == sb["launches"]
    assert np.array_equal(Ca, A @ B)
    A, B = I.problem(720, 360, 540, seed=5, kind="integers")  # <4,3,3>: MK = 12 inputs per row: no collapse
    Ca, sa = _run(F, "alg_433_29", A, B, 2, collapse=True)  # even on request
    assert sa["collapsed"] == 0 and np.array_equal(Ca, A @ B)
    A, B = I.problem(256, 256, 256, seed=6, kind="integers")  # write-once strategy
    Ca, sa = _run(F, "strassen_222_7", A, B, 2, strategy="write_once")
    assert np.array_equal(Ca, A @ B)


# The formation alone for base cases with MK, KN <= 9 (the assembly stays one level per launch):
# (MK)^2 inputs of a position held in one thread's registers
FORM_CASES = [("alg_424_26", 320, 64, 320, "row"), ("hk_class_323_15", 540, 360, 540, "col"),
              ("laderman_class_333_23", 450, 252, 360, "row"), ("direct_223_11", 200, 120, 180, "row")]


@pytest.mark.parametrize("name,P,Q,N,layout", FORM_CASES)
def test_collapsed_formation_equals_separate_and_oracle(name, P, Q, N, layout, monkeypatch):
    monkeypatch.setenv("FMM_COLLAPSE_FORM", "1")  # on request only
    F = _lib()
    A, B = I.problem(P, Q, N, seed=P + Q)
    Cc, sc = _run(F, name, A, B, 2, layout, cse=False, collapse=True)
    Cs, ss = _run(F, name, A, B, 2, layout, cse=False, collapse=False)
    assert sc["collapsed"] == 1 and sc["collapsed_assembly"] == 0
    assert sc["formation_bytes"] < ss["formation_bytes"] and sc["assembly_bytes"] == ss["assembly_bytes"]
    assert np.array_equal(Cc, Cs)  # the oracle's two levels in its order
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(Cc - O.fast(A, B, O.load_alg(F.alg_path(name)), 2))) <= 1e-12 * nrm
    Ai, Bi = I.problem(P, Q, N, seed=3, kind="integers")
    Ci, _ = _run(F, name, Ai, Bi, 2, layout)
    assert np.array_equal(Ci, Ai @ Bi)


@pytest.mark.parametrize("G", [2, 3])
def test_collapsed_formation_shards_sum_to_product(G, monkeypatch):
    monkeypatch.setenv("FMM_COLLAPSE_FORM", "1")
    F = _lib()
    A, B = I.problem(320, 64, 320, seed=8, kind="integers")
    total = np.zeros((320, 320))
    for g in range(G):
        C, st = _run(F, "alg_424_26", A, B, 2, shard_rank=g, shard_count=G)
        assert st["collapsed"] == 1
        total += C
    assert np.array_equal(total, A @ B)


@pytest.mark.parametrize("layout", ["row", "col"])
def test_collapsed_strided_views(layout):
    # padded leading dimensions on A, B and C; nothing outside C is written
    import torch
    F = _lib()
    P, Q, N = 256, 128, 192
    A, B = I.problem(P, Q, N, seed=11, kind="integers")
    if layout == "row":
        Ab = torch.zeros(P, Q + 6, dtype=torch.float64, device="cuda"); Ab[:, 2:Q + 2] = torch.from_numpy(A).cuda()
        Bb = torch.zeros(Q, N + 10, dtype=torch.float64, device="cuda"); Bb[:, 4:N + 4] = torch.from_numpy(B).cuda()
        Cb = torch.full((P, N + 8), 5.0, dtype=torch.float64, device="cuda")
        Av, Bv, Cv = Ab[:, 2:Q + 2], Bb[:, 4:N + 4], Cb[:, 2:N + 2]
    else:
        Ab = torch.zeros(Q, P + 6, dtype=torch.float64, device="cuda"); Ab[:, 2:P + 2] = torch.from_numpy(A.T.copy()).cuda()
        Bb = torch.zeros(N, Q + 10, dtype=torch.float64, device="cuda"); Bb[:, 4:Q + 4] = torch.from_numpy(B.T.copy()).cuda()
        Cb = torch.full((N, P + 8), 5.0, dtype=torch.float64, device="cuda")
        Av, Bv, Cv = Ab[:, 2:P + 2].t(), Bb[:, 4:Q + 4].t(), Cb[:, 2:P + 2].t()
    p = F.Plan(F.load_alg("winograd_class_222_7"), P, Q, N, 2, layout=layout)
    assert p.stats()["collapsed"] == 1
    p.execute(Av, Bv, Cv)
    torch.cuda.synchronize()
    assert np.array_equal(Cv.cpu().numpy(), A @ B)
    rest = Cb.clone()
    if layout == "row":
        rest[:, 2:N + 2] = 5.0
    else:
        rest[:, 2:P + 2] = 5.0
    assert bool((rest == 5.0).all())


# The wide two-level assembly: base cases with MN <= 16 collapse the last two
# levels' assembly only (one warp per output column k2 of W, leaf products staged in shared memory);
# its chains are the oracle's two levels in the oracle's order, so with CSE off it equals the
# one-level-per-launch assembly bit for bit.
WIDE = [("hk_class_323_15", 540, 360, 541, 2, "row"),  # a top-level column strip
        ("alg_424_26", 1008, 240, 960, 2, "row"), ("alg_433_29", 1152, 216, 234, 2, "col"),
        ("laderman_class_333_23", 378, 360, 342, 2, "row"), ("alg_424_26", 128, 32, 2080, 2, "col"),
        ("flip_234_20", 256, 432, 320, 2, "row")]


@pytest.fixture
def wide(monkeypatch):
    monkeypatch.setenv("FMM_WIDE_ASM", "1")  # measured slower than the separate levels: opt-in


@pytest.mark.parametrize("name,P,Q,N,L,layout", WIDE)
def test_wide_assembly_equals_separate_and_oracle(name, P, Q, N, L, layout, wide):
    F = _lib()
    A, B = I.problem(P, Q, N, seed=P + N)
    Cw, sw = _run(F, name, A, B, L, layout, cse=False, collapse=True)
    Cs, ss = _run(F, name, A, B, L, layout, cse=False, collapse=False)
    assert sw["collapsed_assembly"] == 1 and ss["collapsed_assembly"] == 0
    assert sw["add_bytes"] < ss["add_bytes"] and sw["launches"] == ss["launches"] - 1
    assert np.array_equal(Cw, Cs)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(Cw - O.fast(A, B, O.load_alg(F.alg_path(name)), L))) <= 1e-12 * nrm


@pytest.mark.parametrize("G", [2, 5])
def test_wide_assembly_shards_sum_to_product(G, wide):
    F = _lib()
    A, B = I.problem(640, 160, 640, seed=9, kind="integers")
    total = np.zeros((640, 640))
    for g in range(G):
        C, st = _run(F, "alg_424_26", A, B, 2, shard_rank=g, shard_count=G)
        assert st["collapsed_assembly"] == 1
        total += C
    assert np.array_equal(total, A @ B)


def test_wide_assembly_peeled_level_not_collapsed(wide):
    # level L-1 peeled (90 / 2 = 45 is odd, R7b): its strips need the level-(L-1) M, so no collapse
    F = _lib()
    A, B = I.problem(270, 180, 270, seed=5, kind="integers")
    Ca, sa = _run(F, "hk_class_323_15", A, B, 2, collapse=True)
    _, sb = _run(F, "hk_class_323_15", A, B, 2, collapse=False)
    assert sa["collapsed_assembly"] == 0 and sa["launches"] == sb["launches"] and np.array_equal(Ca, A @ B)
