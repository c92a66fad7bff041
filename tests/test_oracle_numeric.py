"""Pins of the numerical oracle (oracle/oracle.c) against things other than itself: brute-force
definitions on tiny inputs, exact integer products (numpy int64 matmul, a library primitive),
the flop-count closed forms of Sec. 2.1, and exactness under quantised inputs.  No GPU."""
import glob
import math
import os

import numpy as np
import pytest

import fmm_inputs as I
from conftest import ALGS, GOLDEN
from oracle import oracle as O

ALG_FILES = sorted(glob.glob(os.path.join(ALGS, "*.txt")))
ALGS_BY_NAME = {os.path.basename(p)[:-4]: O.load_alg(p) for p in ALG_FILES}


def _exact(A, B):
    """Exact product of integer-valued float matrices via int64 (library primitive)."""
    return (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)


def test_classical_matches_brute_force_loops():
    A, B = I.problem(5, 7, 3, seed=1)
    C = O.classical(A, B)
    ref = np.zeros((5, 3))
    for i in range(5):
        for j in range(3):
            s = 0.0
            for q in range(7):
                s = s + A[i, q] * B[q, j]
            ref[i, j] = s
    assert np.array_equal(C, ref)  # same order, same rounding


@pytest.mark.parametrize("layout", ["row", "col"])
def test_classical_integer_exact_both_layouts(layout):
    A, B = I.problem(33, 29, 31, seed=2, kind="integers", layout=layout)
    assert np.array_equal(O.classical(A, B), _exact(A, B))


def test_classical_degenerate_dims():
    A = np.zeros((3, 0)); B = np.zeros((0, 4))
    assert np.array_equal(O.classical(A, B), np.zeros((3, 4)))


# ---- check (c): fast == classical bitwise on integer inputs ----------------------------------
def _cases():
    out = []
    for name, a in ALGS_BY_NAME.items():
        for L in (1, 2):
            out.append((name, L, a.M ** L, a.K ** L, a.N ** L))          # exact base-case powers
            out.append((name, L, 3 * a.M ** L + 1, 2 * a.K ** L + 1, 2 * a.N ** L + 2))  # peeled
    out += [("strassen_222_7", 1, 4, 4, 4), ("strassen_222_7", 2, 4, 4, 4),   # BJ config 1 4x4
            ("strassen_222_7", 1, 5, 5, 5), ("strassen_222_7", 3, 37, 41, 43),
            ("hk_class_323_15", 1, 7, 5, 7), ("hk_class_323_15", 2, 101, 67, 89),
            ("hk_class_323_15", 2, 7, 11, 13), ("laderman_class_333_23", 2, 29, 31, 28)]
    return out


@pytest.mark.parametrize("name,L,P,Q,N", _cases())
def test_fast_equals_classical_bitwise_on_integers(name, L, P, Q, N):
    a = ALGS_BY_NAME[name]
    A, B = I.problem(P, Q, N, seed=L, kind="integers")
    C = O.fast(A, B, a, L)
    assert np.array_equal(C, _exact(A, B))
    assert np.array_equal(C, O.classical(A, B))


def test_fast_col_major_input_equals_row_major():
    a = ALGS_BY_NAME["winograd_class_222_7"]
    Ar, Br = I.problem(36, 20, 28, seed=4)
    Ac, Bc = I.problem(36, 20, 28, seed=4, layout="col")
    assert np.array_equal(O.fast(Ar, Br, a, 2), O.fast(Ac, Bc, a, 2))


def test_fast_degenerate_and_sub_base_case_dims_fall_back_to_classical():
    a = ALGS_BY_NAME["laderman_class_333_23"]
    for (P, Q, N) in [(2, 9, 9), (9, 2, 9), (9, 9, 2), (1, 1, 1)]:
        A, B = I.problem(P, Q, N, seed=3)
        assert np.array_equal(O.fast(A, B, a, 2), O.classical(A, B))


# ---- exactness trick: quantised inputs make every partial sum exact ---------------------------
@pytest.mark.parametrize("name,L,P,Q,N", [
    ("winograd_class_222_7", 2, 256, 256, 256),
    ("hk_class_323_15", 2, 181, 70, 183),
    ("alg_424_26", 2, 160, 40, 163),
    ("laderman_class_333_23", 2, 91, 90, 92),
    ("alg_433_29", 2, 161, 45, 46),
])
def test_fast_exact_on_quantized_inputs(name, L, P, Q, N):
    a = ALGS_BY_NAME[name]
    A, B = I.problem(P, Q, N, seed=5, kind="quantized")
    s = 2.0 ** 11
    exact = _exact(A * s, B * s) / (s * s)
    assert np.array_equal(O.fast(A, B, a, L), exact)


# ---- check (d): error growth within the fixed tolerance (reading R16: parity of the growth
# itself is unpinned by the paper; the gate is BASELINE's 1e-10*|A|_F|B|_F for L <= 3) --------
@pytest.mark.parametrize("name", list(ALGS_BY_NAME))
def test_fast_float_error_within_fixed_tolerance(name):
    a = ALGS_BY_NAME[name]
    P, Q, N = (a.M ** 3 * 3, a.K ** 3 * 3, a.N ** 3 * 3) if a.M * a.K * a.N <= 12 else (a.M ** 2 * 7, a.K ** 2 * 7, a.N ** 2 * 7)
    A, B = I.problem(P, Q, N, seed=6)
    Cc = O.classical(A, B)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    errs = []
    for L in (1, 2, 3) if a.M * a.K * a.N <= 12 else (1, 2):
        e = np.max(np.abs(O.fast(A, B, a, L) - Cc)) / nrm
        errs.append(e)
        assert e <= 1e-10
    assert errs[0] < 1e-15  # rounding-level, far below the gate


# ---- the sampled-entry oracle is bit-identical to the full oracle ------------------------------
@pytest.mark.parametrize("name,L,P,Q,N", [
    ("strassen_222_7", 3, 37, 41, 43), ("winograd_class_222_7", 2, 64, 64, 64),
    ("hk_class_323_15", 2, 101, 67, 89), ("alg_424_26", 2, 70, 9, 66),
    ("laderman_class_333_23", 2, 29, 31, 28), ("alg_433_29", 2, 50, 29, 31)])
def test_fast_entries_bit_identical_to_fast(name, L, P, Q, N):
    a = ALGS_BY_NAME[name]
    A, B = I.problem(P, Q, N, seed=8)
    C = O.fast(A, B, a, L)
    rows, cols = np.meshgrid(np.arange(P), np.arange(N), indexing="ij")
    e = O.fast_entries(A, B, a, L, rows.reshape(-1), cols.reshape(-1))
    assert np.array_equal(e.reshape(P, N), C)
    ce = O.classical_entries(A, B, [0, P - 1, P // 2], [N - 1, 0, N // 3])
    Cc = O.classical(A, B)
    assert np.array_equal(ce, np.array([Cc[0, N - 1], Cc[P - 1, 0], Cc[P // 2, N // 3]]))


# ---- flop counts: Sec. 2.1 closed forms ----------------------------------------
def test_flop_count_closed_forms():
    rows = [ln.split() for ln in open(os.path.join(GOLDEN, "flop_counts.txt")) if ln.strip() and ln[0] != "#"]
    s = ALGS_BY_NAME["strassen_222_7"]
    for kind, n, val in rows:
        n, val = int(n), int(val)
        L = 0 if kind == "classical" else int(math.log2(n))
        assert O.flops(n, n, n, s, L) == val
    for k in range(0, 7):
        n = 2 ** k
        assert O.flops(n, n, n, s, 0) == 2 * n ** 3 - n ** 2
        assert O.flops(n, n, n, s, k) == round(7 * n ** math.log2(7) - 6 * n ** 2)


def test_flop_count_peeled_and_scaled_by_hand():
    # the branches the closed forms above do not reach, counted by hand from the paper's
    # operation rules: a classical p x q x n product costs p n (2q - 1); a chain of k
    # nonzero coefficients costs k - 1 additions per element, and a non-unit coefficient one multiply
    # per element ("inactive multiplies"); peeling per S:287-295 (reading R7)
    import dataclasses
    from fractions import Fraction as Fr
    s = ALGS_BY_NAME["strassen_222_7"]
    # Strassen's 18 block additions: 5 forming S (U), 5 forming T (V), 8 forming C (W)
    assert sum(sum(1 for v in col if v != 0) - 1 for col in zip(*s.U)) == 5
    assert sum(sum(1 for v in col if v != 0) - 1 for col in zip(*s.V)) == 5
    assert sum(sum(1 for v in row if v != 0) - 1 for row in s.W) == 8
    # 5 x 5 x 5, one step: core 4 x 4 x 4 with 2 x 2 blocks
    core = 5 * 4 + 5 * 4 + 7 * (2 * 2 * (2 * 2 - 1)) + 8 * 4       # S, T, 7 leaves of 12 flops, C = 156
    fix_a = 4 * 4 * (2 * 1 - 1) + 4 * 4                             # (a) C'[0:4,0:4] += A[:,4:5] B[4:5,:]
    fix_b = 1 * 5 * (2 * 5 - 1)                                     # (b) the last row of C, classical
    fix_c = 4 * 1 * (2 * 5 - 1)                                     # (c) the last column of the first 4 rows
    assert (core, fix_a, fix_b, fix_c) == (156, 32, 45, 36)
    assert O.flops(5, 5, 5, s, 1) == core + fix_a + fix_b + fix_c == 269
    # rational-scaled column: U column 0 (S_1 = A11 + A22) times 2, W column 0 (M_1 in C11 and C22)
    # times 1/2 -- still exact (Brent), and each scaled coefficient costs one multiply per element
    U = [[v * (2 if r == 0 else 1) for r, v in enumerate(row)] for row in s.U]
    W = [[v * (Fr(1, 2) if r == 0 else 1) for r, v in enumerate(row)] for row in s.W]
    t = dataclasses.replace(s, U=U, W=W)
    assert O.brent_residuals(t) == 0
    # S_1: 1 addition + 2 multiplies per element instead of 1 addition: +2 x 4; C11, C22: +1 x 4 each
    assert O.flops(4, 4, 4, t, 1) == 156 + 2 * 4 + 2 * 4 == 172
    # and a base case smaller than the problem in one dimension only: classical at that level (R10/R18)
    assert O.flops(1, 7, 9, s, 2) == 1 * 9 * (2 * 7 - 1)


# ---- check (d): error growth within the bound derived from (U, V, W) ------------
def _higham_strassen(n, n0):
    """Higham, Accuracy and Stability of Numerical Algorithms (cited at P:80), the Strassen bound:
    ||C - fl(C)||_max <= [(n/n0)^log2(12) (n0^2 + 5 n0) - 5 n] u ||A||_max ||B||_max + O(u^2)."""
    return ((n / n0) ** np.log2(12) * (n0 * n0 + 5 * n0) - 5 * n) * 2.0 ** -53


@pytest.mark.parametrize("n0", [16, 64, 256])
@pytest.mark.parametrize("L", [1, 2, 3])
def test_error_bound_reduces_to_highams_strassen_bound(n0, L):
    a = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    n = n0 * 2 ** L
    ours, textbook = O.error_bound(a, n, L), _higham_strassen(n, n0)
    # the leading terms agree; ours counts left-to-right chains (3 additions in C11 / C22), so its
    # O(n0) lower-order term is slightly larger, never smaller
    assert 1.0 <= ours / textbook < 1.05


def test_error_bound_classical_leaf():
    a = O.load_alg(os.path.join(ALGS, "strassen_222_7.txt"))
    for q in (1, 7, 1000):
        assert O.error_bound(a, q, 0, 2.0, 3.0) == pytest.approx(q * 2.0 ** -53 / (1 - q * 2.0 ** -53) * q * 6.0)


def _exact(A, B):
    return (A.astype(np.longdouble) @ B.astype(np.longdouble))


@pytest.mark.parametrize("name", sorted(ALGS_BY_NAME))
@pytest.mark.parametrize("L", [1, 2])
def test_fast_error_within_derived_bound(name, L):
    alg = ALGS_BY_NAME[name]
    P, Q, N = alg.M ** L * 12, alg.K ** L * 16, alg.N ** L * 12
    A, B = I.problem(P, Q, N, seed=31 + L)
    err = float(np.max(np.abs(O.fast(A, B, alg, L).astype(np.longdouble) - _exact(A, B))))
    bound = O.error_bound(alg, Q, L, float(np.abs(A).max()), float(np.abs(B).max()))
    assert err <= bound
    assert bound <= 1e-10 * np.linalg.norm(A) * np.linalg.norm(B)  # consistent with BJ's gate


def test_error_bound_catches_a_broken_algorithm():
    alg = O.load_alg(os.path.join(ALGS, "winograd_class_222_7.txt"))
    bad = O.Alg(alg.M, alg.K, alg.N, alg.R, [list(r) for r in alg.U], [list(r) for r in alg.V],
                [list(r) for r in alg.W], name="broken")
    r = next(r for r in range(alg.R) if bad.W[0][r] != 0)
    bad.W[0][r] = -bad.W[0][r]  # one flipped sign
    A, B = I.problem(64, 64, 64, seed=5)
    err = float(np.max(np.abs(O.fast(A, B, bad, 2).astype(np.longdouble) - _exact(A, B))))
    assert err > O.error_bound(alg, 64, 2, float(np.abs(A).max()), float(np.abs(B).max()))


# ---- addition-chain traffic per recursion node (Sec. 3.2) ----------------------------
@pytest.mark.parametrize("name", sorted(ALGS_BY_NAME))
def test_addition_traffic_matches_the_papers_closed_forms(name):
    # the chain-by-chain count against the paper's closed forms
    a = ALGS_BY_NAME[name]
    nu, nv, nw = a.nnz()
    nnz, R, MN = nu + nv + nw, a.R, a.M * a.N
    single = sum(1 for X in (a.U, a.V) for r in range(R) if sum(1 for row in X if row[r] != 0) == 1)
    assert O.addition_traffic(a, "pairwise") == (2 * nnz - 2 * R - MN, nnz)
    rw, ww = O.addition_traffic(a, "write_once")
    assert rw == nnz and ww == 2 * R + MN - single and ww <= 2 * R + MN
    rs, ws = O.addition_traffic(a, "streaming")
    every_block_used = all(any(v != 0 for v in row) for X in (a.U, a.V) for row in X)
    assert every_block_used and rs == a.M * a.K + a.K * a.N + R
    assert ws == ww
    # aliasing the one-term U / V chains removes exactly one read (and, pairwise, one write) each
    assert O.addition_traffic(a, "pairwise", True) == (2 * nnz - 2 * R - MN - single, nnz - single)
    assert O.addition_traffic(a, "write_once", True) == (nnz - single, ww)


def test_addition_traffic_strassen_and_winograd_values():
    # SURVEY 8(d)'s verified counts (paper convention, then with singleton chains aliased)
    s, w = ALGS_BY_NAME["strassen_222_7"], ALGS_BY_NAME["winograd_class_222_7"]
    assert [O.addition_traffic(s, k) for k in ("pairwise", "write_once", "streaming")] == [(54, 36), (36, 14), (15, 14)]
    assert [O.addition_traffic(w, k) for k in ("pairwise", "write_once", "streaming")] == [(66, 42), (42, 12), (15, 12)]
    assert O.addition_traffic(s, "write_once", True) == (32, 14) and O.addition_traffic(w, "write_once", True) == (36, 12)
