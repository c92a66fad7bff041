"""Pins of the oracle's exact algebra against what the paper prints and what mathematics fixes.
No GPU.  P:<line> = /root/reference/PAPER.md line."""
import glob
import itertools
import math
import os
import random
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ALGS, GOLDEN
from oracle import oracle as O

ALG_FILES = sorted(glob.glob(os.path.join(ALGS, "*.txt")))


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


# ---- the matmul tensor -------------------------------------------------
def test_tensor_222_frontal_slices_match_paper():
    lines = _golden("tensor_222_slices.txt")
    T = O.matmul_tensor(2, 2, 2)
    slices, cur = [], None
    for ln in lines:
        if ln.startswith("slice"):
            cur = []
            slices.append(cur)
        else:
            cur.append([int(v) for v in ln.split()])
    assert len(slices) == 4
    for k in range(4):
        assert np.array_equal(T[:, :, k], np.array(slices[k])), f"slice {k+1}"


def test_tensor_T3_worked_example_gives_C21():
    # T_3 x1 vec(A) x2 vec(B) = A21*B11 + A22*B21 = C21
    T = O.matmul_tensor(2, 2, 2)
    rng = random.Random(3)
    for _ in range(20):
        a = [rng.randint(-9, 9) for _ in range(4)]
        b = [rng.randint(-9, 9) for _ in range(4)]
        z = O.contract(T, a, b)
        assert z[2] == a[2] * b[0] + a[3] * b[2]


@pytest.mark.parametrize("M,K,N", list(itertools.product(range(1, 5), repeat=3)))
def test_tensor_has_MKN_nonzeros_and_contracts_to_matmul(M, K, N):
    T = O.matmul_tensor(M, K, N)
    assert T.sum() == M * K * N  # P:414 "MKN non-zeros"
    assert set(np.unique(T)) <= {0, 1}
    rng = np.random.default_rng(M * 100 + K * 10 + N)
    A = rng.integers(-5, 6, size=(M, K))
    B = rng.integers(-5, 6, size=(K, N))
    z = O.contract(T, list(A.reshape(-1)), list(B.reshape(-1)))  # row-major vec
    assert np.array_equal(np.array(z).reshape(M, N), A @ B)


# ---- Strassen -----------------------------------------------------------
def _formula_alg(lines):
    """Build U,V,W from 'S1 = A11 + A22' style formulas."""
    U = [[Fraction(0)] * 7 for _ in range(4)]
    V = [[Fraction(0)] * 7 for _ in range(4)]
    W = [[Fraction(0)] * 7 for _ in range(4)]
    for ln in lines:
        lhs, rhs = [s.strip() for s in ln.split("=")]
        terms = re.findall(r"([+-]?)\s*([ABM])(\d+)", rhs)
        for sign, kind, idx in terms:
            c = Fraction(-1 if sign == "-" else 1)
            if lhs[0] in "ST":
                r = int(lhs[1:]) - 1
                row = (int(idx[0]) - 1) * 2 + (int(idx[1]) - 1)
                (U if lhs[0] == "S" else V)[row][r] = c
            else:
                row = (int(lhs[1]) - 1) * 2 + (int(lhs[2]) - 1)
                W[row][int(idx) - 1] = c
    return O.Alg(2, 2, 2, 7, U, V, W)


def test_strassen_sec21_formulas_are_exact_and_match_algs_file():
    f = _formula_alg(_golden("strassen_sec21.txt"))
    assert O.brent_residuals(f) == 0
    s = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    assert (s.U, s.V, s.W) == (f.U, f.V, f.W)


def test_strassen_printed_UV_correct_printed_W_garbled():
    printed = O.parse_alg_text("\n".join(_golden("strassen_printed.txt")))
    f = _formula_alg(_golden("strassen_sec21.txt"))
    assert printed.U == f.U and printed.V == f.V  # P:384-395 agree with Sec. 2.1
    assert O.brent_residuals(printed) > 0           # P:396-401 fails (reading R1)


def test_strassen_scalar_C11_example():
    # S1 = a11 + a22, T1 = b11 + b22, C11 = M1 + M4 - M5 + M7
    s = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    rng = random.Random(7)
    for _ in range(50):
        a = [Fraction(rng.randint(-20, 20)) for _ in range(4)]
        b = [Fraction(rng.randint(-20, 20)) for _ in range(4)]
        S = [sum(s.U[i][r] * a[i] for i in range(4)) for r in range(7)]
        T = [sum(s.V[j][r] * b[j] for j in range(4)) for r in range(7)]
        Mv = [S[r] * T[r] for r in range(7)]
        assert S[0] == a[0] + a[3] and T[0] == b[0] + b[3]
        c11 = Mv[0] + Mv[3] - Mv[4] + Mv[6]
        assert c11 == a[0] * b[0] + a[1] * b[2]
        assert [sum(s.W[k][r] * Mv[r] for r in range(7)) for k in range(4)] == \
            [a[0] * b[0] + a[1] * b[2], a[0] * b[1] + a[1] * b[3], a[2] * b[0] + a[3] * b[2], a[2] * b[1] + a[3] * b[3]]


# ---- Brent equations for every algorithm ------------------------------------
@pytest.mark.parametrize("path", ALG_FILES, ids=os.path.basename)
def test_brent_exact_all_files(path):
    a = O.load_alg(path)
    assert O.brent_residuals(a) == 0
    assert all(v in (-1, 0, 1) for X in (a.U, a.V, a.W) for row in X for v in row)


@pytest.mark.parametrize("path", ALG_FILES, ids=os.path.basename)
def test_brent_detects_any_single_coefficient_error(path):
    a = O.load_alg(path)
    rng = random.Random(11)
    for _ in range(12):
        which = rng.choice("UVW")
        X = [list(r) for r in getattr(a, which)]
        i = rng.randrange(len(X)); r = rng.randrange(a.R)
        X[i][r] = X[i][r] + rng.choice([-1, 1])  # a dropped/added term or a wrong sign
        b = O.Alg(a.M, a.K, a.N, a.R, *(X if w == which else getattr(a, w) for w in "UVW"))
        assert O.brent_residuals(b) > 0


@pytest.mark.parametrize("M,K,N", [(1, 1, 1), (2, 2, 2), (2, 3, 4), (3, 2, 3), (4, 3, 2)])
def test_classical_decomposition_exact(M, K, N):
    assert O.brent_residuals(O.classical_alg(M, K, N)) == 0


# ---- Props 1-3 ---------------------------------------------------------------------
@pytest.mark.parametrize("path", ALG_FILES, ids=os.path.basename)
def test_prop1_prop2_generate_all_six_permutations(path):
    a = O.load_alg(path)
    seen = {}
    frontier = [a]
    while frontier:
        x = frontier.pop()
        key = (x.M, x.K, x.N)
        if key in seen:
            continue
        assert O.brent_residuals(x) == 0, key
        seen[key] = x
        frontier += [O.prop1(x), O.prop2(x)]
    assert set(seen) == set(itertools.permutations((a.M, a.K, a.N)))


def test_prop3_perm_scale_and_basis_change():
    s = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    rng = random.Random(5)
    perm = list(range(7)); rng.shuffle(perm)
    dx = [Fraction(rng.choice([1, -1, 2])) for _ in range(7)]
    dy = [Fraction(rng.choice([1, -1, 3])) for _ in range(7)]
    dz = [1 / (dx[r] * dy[r]) for r in range(7)]
    assert O.brent_residuals(O.prop3_perm_scale(s, perm, dx, dy, dz)) == 0
    F = lambda m: [[Fraction(v) for v in r] for r in m]
    X, Y, Z = F([[2, 1], [1, 1]]), F([[1, -1], [0, 1]]), F([[0, 1], [1, 3]])
    assert O.brent_residuals(O.prop3_basis(s, X, Y, Z)) == 0


def test_winograd_class_is_prop3_image_of_strassen():
    s = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    w = O.load_alg(os.path.join(ALGS, "winograd_class_222_7.txt"))
    F = lambda m: [[Fraction(v) for v in r] for r in m]
    t = O.prop3_basis(s, F([[-1, -1], [-1, 0]]), F([[-1, 0], [-1, 1]]), F([[-1, 0], [0, -1]]))
    assert (t.U, t.V, t.W) == (w.U, w.V, w.W)
    assert w.nnz() == (14, 14, 14)


# ---- Table 2 -----------------------------------------------------------------------
def test_table2_speedups_and_our_ranks():
    rows = [list(map(int, ln.split())) for ln in _golden("table2.txt")]
    for M, K, N, R, classical, pct in rows:
        mkn = M * K * N
        if (M, K, N) == (3, 3, 3):
            assert classical == 26 and mkn == 27  # printed typo, reading R4
        else:
            assert classical == mkn
        assert round(100 * (mkn / R - 1)) == pct
    ranks = {tuple(sorted((M, K, N))): R for M, K, N, R, _, _ in rows}
    above = {"flip_344_39.txt": 1}  # our <3,4,4> is one multiplication above Table 2's 38 (DESIGN f2)
    for path in ALG_FILES:
        a = O.load_alg(path)
        # the paper's rank reached (or, for the files listed, missed by the stated amount)
        assert a.R == ranks[tuple(sorted((a.M, a.K, a.N)))] + above.get(os.path.basename(path), 0), path
