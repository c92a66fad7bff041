"""Shape matching and the cutoff rule: Prop. 1/2 permutations of every
algorithm (fmm_alg_permute), the host cost model (fmm_plan_predict) and the selector (fmm_select).

CPU: every permutation has the permuted base case and passes the library's exact Brent re-check;
independently, the oracle's own Props. 1/2 composed the same way are exact with the same shapes;
the cost model is consistent with plain facts (classical time ~ 2PQN / peak, the recursion stops
below the base case, Strassen beats classical at 8192^3 and loses at 128^3); the selector's answer
is never predicted slower than any candidate it saw.
GPU: permuted algorithms multiply integer matrices exactly; the selected plans meet the tolerance.
"""
import glob
import os

import numpy as np
import pytest

import fmm_inputs as I
from conftest import ALGS
from oracle import oracle as O

NAMES = [os.path.basename(p)[:-4] for p in sorted(glob.glob(os.path.join(ALGS, "*.txt")))]
SHAPE = {0: "MKN", 1: "NKM", 2: "NMK", 3: "KNM", 4: "KMN", 5: "MNK"}


def _lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


@pytest.mark.parametrize("name", NAMES)
def test_permutation_shapes_and_exactness(name):
    F = _lib()
    a = F.load_alg(name)
    dims = {"M": a.M, "K": a.K, "N": a.N}
    for p in range(6):
        b = a.permute(p)  # the library re-validates the Brent equations exactly (FMM_E_NOT_EXACT otherwise)
        want = [dims[c] for c in SHAPE[p]]
        assert [b.M, b.K, b.N] == want and b.R == a.R
        assert sorted(b.nnz) == sorted(a.nnz)  # permutations only move coefficients


@pytest.mark.parametrize("name", ["hk_class_323_15", "alg_433_29", "direct_225_18"])
def test_permutation_matches_oracle_propositions(name):
    # the oracle's Props. 1/2 (oracle/oracle.py, exact Fractions) give the same base cases and
    # exact algorithms; compose them the way fmm_alg_permute documents
    o = O.load_alg(os.path.join(ALGS, name + ".txt"))
    seq = {0: [], 1: ["p1"], 2: ["p2"], 3: ["p2", "p2"], 4: ["p2", "p1"], 5: ["p2", "p2", "p1"]}
    for p, ops in seq.items():
        b = o
        for op in ops:
            b = O.prop1(b) if op == "p1" else O.prop2(b)
        assert O.brent_residuals(b) == 0
        want = {"M": o.M, "K": o.K, "N": o.N}
        assert [b.M, b.K, b.N] == [want[c] for c in SHAPE[p]]


def test_cost_model_classical_and_cutoff():
    F = _lib()
    s = F.load_alg("strassen_222_7")
    # L = 0 is one classical DMMA GEMM: within 10 % of 2PQN at the model's 148 x 245 GFLOP/s
    for n in (4096, 8192):
        t = s.predict_ms(n, n, n, 0) * 1e-3
        assert abs(t - 2.0 * n ** 3 / (148 * 245e9)) / t < 0.10
    # the recursion stops below the base case: levels beyond it cost the same as the last taken
    assert s.predict_ms(5, 5, 5, 8) == s.predict_ms(5, 5, 5, 2)
    # large square problems: one Strassen level beats classical (Table 2: 14 % fewer multiplies)
    assert s.predict_ms(8192, 8192, 8192, 1) < s.predict_ms(8192, 8192, 8192, 0)
    # tiny problems: classical wins (the paper's cutoff, Sec. 3.4)
    assert s.predict_ms(128, 128, 128, 0) < s.predict_ms(128, 128, 128, 1)


@pytest.mark.parametrize("shape", [(256, 256, 256), (8192, 8192, 8192), (12000, 1800, 12000), (18000, 3600, 3600),
                                   (3000, 3000, 900)])
def test_select_is_the_predicted_minimum(shape):
    F = _lib()
    P, Q, N = shape
    algs = [F.load_alg(n) for n in NAMES]
    sel, L, ms = F.select(algs, P, Q, N, 3)
    classical = algs[0].predict_ms(P, Q, N, 0)
    assert ms <= classical * (1 + 1e-9)
    if sel is None:
        assert L == 0 and abs(ms - classical) < 1e-9
    else:
        assert 1 <= L <= 3 and abs(sel.predict_ms(P, Q, N, L) - ms) < 1e-6 * ms
    for a in algs:  # nothing it saw is predicted faster
        for p in range(6):
            b = a.permute(p)
            for LL in range(1, 4):
                assert b.predict_ms(P, Q, N, LL) >= ms * (1 - 1e-9)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["hk_class_323_15", "alg_433_29", "direct_223_11"])
@pytest.mark.parametrize("perm", range(6))
def test_permuted_algorithms_multiply_correctly(name, perm):
    import torch
    F = _lib()
    a = F.load_alg(name).permute(perm)
    P, Q, N = 2 * a.M ** 2 + 1, 3 * a.K ** 2 + 2, 2 * a.N ** 2 + 1
    A, B = I.problem(P, Q, N, seed=perm, kind="integers")
    p = F.Plan(a, P, Q, N, 2)
    C = p.execute(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    assert np.array_equal(C, A @ B)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(1536, 1536, 1536), (2400, 300, 2400), (3600, 720, 720)])
def test_selected_plan_parity(shape):
    import torch
    F = _lib()
    P, Q, N = shape
    sel, L, _ = F.select([F.load_alg(n) for n in NAMES], P, Q, N, 2)
    A, B = I.problem(P, Q, N, seed=P)
    if sel is None:
        C = F.dgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
        assert np.max(np.abs(C - O.classical(A, B))) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(B)
        return
    p = F.Plan(sel, P, Q, N, L)
    C = p.execute(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(C - O.classical(A, B))) <= 1e-10 * nrm


@pytest.mark.gpu
@pytest.mark.parametrize("name,P,Q,N,layout", [("strassen_222_7", 2048, 2048, 2048, "row"), ("alg_424_26", 3000, 600, 3000, "col"),
                                               ("strassen_222_7", 200, 200, 200, "row")])
def test_automatic_levels(name, P, Q, N, layout):
    # levels = -1: the plan takes the cost model's fastest L <= 4, and still multiplies exactly
    import torch
    F = _lib()
    a = F.load_alg(name)
    preds = [a.predict_ms(P, Q, N, L, layout) for L in range(5)]
    p = F.Plan(a, P, Q, N, -1, layout=layout)
    assert p.stats()["levels"] == int(np.argmin(preds)) or preds[int(p.stats()["levels"])] <= min(preds) * (1 + 1e-9)
    A, B = I.problem(P, Q, N, seed=7, kind="integers")
    dev = (lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()) if layout == "row" else \
          (lambda x: torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t())
    C = p.execute(dev(A), dev(B)).cpu().numpy()
    assert np.array_equal(C, A @ B)
