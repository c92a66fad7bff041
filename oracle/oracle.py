"""ORACLE — TEST INFRASTRUCTURE ONLY (arXiv 1409.2908, /root/reference/PAPER.md = P:<line>).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  It shares no code with the CUDA path in paper_1409_2908_b200/ and neither
side imports the other; the only common module is fmm_inputs (seeded input generators, no
arithmetic of the method).

Contents
  * exact algebra (Python fractions.Fraction, no floating point):
      matmul_tensor(M,K,N)        the <M,K,N> tensor from the index conditions of P:415-421
      brent_residuals(alg)        sum_r u_ir v_jr w_kr - T_ijk over all (i,j,k)
      prop1 / prop2 / prop3       the transformations of Props 1-3 (Prop 3 in the
                                  row-major reading R2 of DESIGN.md)
      classical_alg(M,K,N)        the rank-MKN classical algorithm (P:224-233 generalised)
      contract(T, a, b)           z_k = sum_ij T_ijk a_i b_j  (Eq. conventional)
  * the algorithm file parser of the S:190 text format (independent of the library's parser)
  * numerical oracle (C, liboracle.so, -ffp-contract=off):
      classical(A, B)             the definition C_ij = sum_q A_iq B_qj
      fast(A, B, alg, L)          the recursive evaluation with peeling
      fast_entries(A, B, alg, L, rows, cols)  sampled entries of exactly fast(...)
      flops(P,Q,N, alg, L)        operation count of fast(...)
  * addition_traffic(alg, strategy, alias_singletons)  sub-block reads / writes of one recursion
                                  node's addition chains, counted chain by chain for the pairwise,
                                  write-once and streaming implementations
  * error_bound(alg, Q, L, a, b)  a worst-case forward error bound on max|fl(C) - C| derived from
                                  (U, V, W) ("theoretical bounds can be derived from each
                                  algorithm's <U,V,W> representation"); pins check (d) of SURVEY 8(c)
                                  in place of the empirical growth figure the paper does not state.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from fractions import Fraction
from typing import List, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


# --------------------------------------------------------------------------------------------
# exact algebra
# --------------------------------------------------------------------------------------------
@dataclass
class Alg:
    """A bilinear algorithm <U,V,W> for base case <M,K,N> with rank R.

    U is MK x R, V is KN x R, W is MN x R, entries exact Fractions, rows in the paper's
    row-major block vectorisation: A-block (a,b) is row a*K+b, B-block (b,c) is row
    b*N+c, C-block (a,c) is row a*N+c.
    """
    M: int
    K: int
    N: int
    R: int
    U: List[List[Fraction]]
    V: List[List[Fraction]]
    W: List[List[Fraction]]
    name: str = ""

    def as_float(self):
        f = lambda X: np.array([[float(v) for v in row] for row in X], dtype=np.float64)
        return f(self.U), f(self.V), f(self.W)

    def nnz(self):
        c = lambda X: sum(1 for row in X for v in row if v != 0)
        return c(self.U), c(self.V), c(self.W)


def tensor_entry(M: int, K: int, N: int, i: int, j: int, k: int) -> int:
    """T_ijk for <M,K,N>, 0-based indices, from the 1-indexed conditions of P:415-421:
    (i-1) mod K = floor((j-1)/N);  (j-1) mod N = (k-1) mod N;  floor((i-1)/K) = floor((k-1)/N).
    With 0-based i,j,k the '-1' shifts disappear."""
    return int(i % K == j // N and j % N == k % N and i // K == k // N)


def matmul_tensor(M: int, K: int, N: int) -> np.ndarray:
    """Dense MK x KN x MN 0/1 tensor."""
    T = np.zeros((M * K, K * N, M * N), dtype=np.int64)
    for i in range(M * K):
        for j in range(K * N):
            for k in range(M * N):
                T[i, j, k] = tensor_entry(M, K, N, i, j, k)
    return T


def contract(T: np.ndarray, a: Sequence, b: Sequence) -> list:
    """z_k = sum_i sum_j T_ijk a_i b_j  (Eq. conventional), exact on Python objects."""
    I, J, K = T.shape
    return [sum(T[i, j, k] * a[i] * b[j] for i in range(I) for j in range(J) if T[i, j, k]) for k in range(K)]


def brent_residuals(alg: Alg) -> int:
    """Number of (i,j,k) where sum_r u_ir v_jr w_kr != T_ijk, in exact rational arithmetic
    (the (MKN)^2 polynomial equations of, Eq. lowrank)."""
    M, K, N, R = alg.M, alg.K, alg.N, alg.R
    bad = 0
    for i in range(M * K):
        ui = alg.U[i]
        for j in range(K * N):
            vj = alg.V[j]
            uv = [ui[r] * vj[r] for r in range(R)]
            for k in range(M * N):
                wk = alg.W[k]
                s = sum((uv[r] * wk[r] for r in range(R) if uv[r] != 0 and wk[r] != 0), Fraction(0))
                if s != tensor_entry(M, K, N, i, j, k):
                    bad += 1
    return bad


def classical_alg(M: int, K: int, N: int) -> Alg:
    """The classical algorithm as a rank-MKN decomposition: one product A_ab * B_bc per
    (a,b,c), added into C_ac (P:224-233 for <2,2,2>)."""
    R = M * K * N
    U = [[Fraction(0)] * R for _ in range(M * K)]
    V = [[Fraction(0)] * R for _ in range(K * N)]
    W = [[Fraction(0)] * R for _ in range(M * N)]
    r = 0
    for a in range(M):
        for b in range(K):
            for c in range(N):
                U[a * K + b][r] = Fraction(1)
                V[b * N + c][r] = Fraction(1)
                W[a * N + c][r] = Fraction(1)
                r += 1
    return Alg(M, K, N, R, U, V, W, name=f"classical_{M}{K}{N}")


def _perm_rows(X, I, J):
    """P_{IxJ} X: P_{IxJ} vec(A) = vec(A^T) for an I x J matrix A.
    Row (c*I + a) of the result is row (a*J + c) of X."""
    out = [None] * (I * J)
    for a in range(I):
        for c in range(J):
            out[c * I + a] = list(X[a * J + c])
    return out


def prop1(alg: Alg) -> Alg:
    """Prop. 1: <P_{KxN} V, P_{MxK} U, P_{MxN} W> is an algorithm for <N,K,M>."""
    M, K, N = alg.M, alg.K, alg.N
    return Alg(N, K, M, alg.R, _perm_rows(alg.V, K, N), _perm_rows(alg.U, M, K), _perm_rows(alg.W, M, N),
               name=alg.name + "^T")


def prop2(alg: Alg) -> Alg:
    """Prop. 2: <P_{MxN} W, U, P_{KxN} V> is an algorithm for <N,M,K>."""
    M, K, N = alg.M, alg.K, alg.N
    return Alg(N, M, K, alg.R, _perm_rows(alg.W, M, N), [list(r) for r in alg.U], _perm_rows(alg.V, K, N),
               name=alg.name + "^cyc")


def _matmul(X, Y):
    return [[sum((X[i][t] * Y[t][j] for t in range(len(Y))), Fraction(0)) for j in range(len(Y[0]))]
            for i in range(len(X))]


def _kron(X, Y):
    return [[X[i // len(Y)][j // len(Y[0])] * Y[i % len(Y)][j % len(Y[0])]
             for j in range(len(X[0]) * len(Y[0]))] for i in range(len(X) * len(Y))]


def _inv(X):
    n = len(X)
    A = [[Fraction(v) for v in row] + [Fraction(int(i == j)) for j in range(n)] for i, row in enumerate(X)]
    for col in range(n):
        piv = next(r for r in range(col, n) if A[r][col] != 0)
        A[col], A[piv] = A[piv], A[col]
        pv = A[col][col]
        A[col] = [v / pv for v in A[col]]
        for r in range(n):
            if r != col and A[r][col] != 0:
                f = A[r][col]
                A[r] = [x - f * y for x, y in zip(A[r], A[col])]
    return [row[n:] for row in A]


def _T(X):
    return [list(r) for r in zip(*X)]


def prop3_basis(alg: Alg, X, Y, Z) -> Alg:
    """Prop. 3 basis change, row-major-vec reading R2 of DESIGN.md:
    U' = (X (x) Y) U, V' = (Y^{-T} (x) Z) V, W' = (X^{-T} (x) Z^{-T}) W, for nonsingular
    X (MxM), Y (KxK), Z (NxN).  With row-major vec, (X (x) Y) vec(A) = vec(X A Y^T), so the new
    algorithm evaluates the old one on X^T A Y and Y^{-1} B Z and maps the product back with
    X^{-T} (.) Z^{-1}."""
    Xi, Yi, Zi = _T(_inv(X)), _T(_inv(Y)), _T(_inv(Z))
    U = _matmul(_kron(X, Y), alg.U)
    V = _matmul(_kron(Yi, Z), alg.V)
    W = _matmul(_kron(Xi, Zi), alg.W)
    return Alg(alg.M, alg.K, alg.N, alg.R, U, V, W, name=alg.name + "^basis")


def prop3_perm_scale(alg: Alg, perm: Sequence[int], dx, dy, dz) -> Alg:
    """Prop. 3: <U P, V P, W P> for a column permutation P and <U Dx, V Dy, W Dz>
    with Dx Dy Dz = I."""
    R = alg.R
    assert all(Fraction(dx[r]) * dy[r] * dz[r] == 1 for r in range(R))
    f = lambda X, d: [[Fraction(row[perm[r]]) * d[r] for r in range(R)] for row in X]
    return Alg(alg.M, alg.K, alg.N, R, f(alg.U, dx), f(alg.V, dy), f(alg.W, dz), name=alg.name + "^ps")


# --------------------------------------------------------------------------------------------
# file format: '#' comments; "M K N R exact"; MK rows of U; blank; KN rows of V; blank;
# MN rows of W.  Entries are integers or rationals p/q.
# --------------------------------------------------------------------------------------------
def parse_alg_text(text: str, name: str = "") -> Alg:
    rows = []
    header = None
    for ln in text.splitlines():
        s = ln.split("#", 1)[0].strip()
        if not s:
            continue
        toks = s.split()
        if header is None:
            if len(toks) < 4:
                raise ValueError("bad header line")
            header = [int(t) for t in toks[:4]]
            if len(toks) > 4 and toks[4] != "exact":
                raise ValueError("only exact algorithms are supported")
            continue
        rows.append([Fraction(t) for t in toks])
    M, K, N, R = header
    if len(rows) != M * K + K * N + M * N or any(len(r) != R for r in rows):
        raise ValueError(f"expected {M*K}+{K*N}+{M*N} rows of {R} entries")
    U = rows[:M * K]
    V = rows[M * K:M * K + K * N]
    W = rows[M * K + K * N:]
    return Alg(M, K, N, R, U, V, W, name=name)


def load_alg(path: str) -> Alg:
    with open(path) as f:
        return parse_alg_text(f.read(), name=os.path.splitext(os.path.basename(path))[0])


# --------------------------------------------------------------------------------------------
# numerical oracle (C)
# --------------------------------------------------------------------------------------------
def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, OpenMP, no FMA contraction)."""
    import fcntl
    stale = lambda: not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC)  # noqa: E731
    if not (force or stale()):
        return _SO
    # concurrent builders (one per rank) take turns; the .so is replaced atomically
    with open(_SO + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if force or stale():
            tmp = f"{_SO}.{os.getpid()}.tmp"
            subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                                   "-shared", "-o", tmp, _SRC])
            os.replace(tmp, _SO)
        fcntl.flock(lk, fcntl.LOCK_UN)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, dp, ip = ctypes.c_int64, ctypes.POINTER(ctypes.c_double), ctypes.c_int
        lib.oracle_classical.argtypes = [i64, i64, i64, dp, i64, i64, dp, i64, i64, dp, i64, i64]
        lib.oracle_fast.argtypes = [i64, i64, i64, dp, i64, i64, dp, i64, i64, dp, i64, i64,
                                    ip, ip, ip, ip, dp, dp, dp, ip]
        lib.oracle_fast_entries.argtypes = [i64, i64, i64, dp, i64, i64, dp, i64, i64,
                                            ip, ip, ip, ip, dp, dp, dp, ip, i64,
                                            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64), dp]
        lib.oracle_flops.argtypes = [i64, i64, i64, ip, ip, ip, ip, dp, dp, dp, ip]
        lib.oracle_flops.restype = ctypes.c_double
        _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _strides(a: np.ndarray):
    assert a.dtype == np.float64 and a.ndim == 2
    return a.strides[0] // 8, a.strides[1] // 8


def classical(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """C = A*B by the definition, q ascending, fp64, no FMA."""
    P, Q = A.shape
    Q2, Nc = B.shape
    assert Q == Q2
    C = np.empty((P, Nc), dtype=np.float64)
    ars, acs = _strides(A); brs, bcs = _strides(B)
    _L().oracle_classical(P, Q, Nc, _dp(A), ars, acs, _dp(B), brs, bcs, _dp(C), Nc, 1)
    return C


def _alg_arrays(alg: Alg):
    U, V, W = alg.as_float()
    return np.ascontiguousarray(U), np.ascontiguousarray(V), np.ascontiguousarray(W)


def fast(A: np.ndarray, B: np.ndarray, alg: Alg, L: int) -> np.ndarray:
    """Recursive fast product of the logical matrices A (P x Q) and B (Q x N), L steps."""
    P, Q = A.shape
    Q2, Nc = B.shape
    assert Q == Q2
    U, V, W = _alg_arrays(alg)
    C = np.empty((P, Nc), dtype=np.float64)
    ars, acs = _strides(A); brs, bcs = _strides(B)
    _L().oracle_fast(P, Q, Nc, _dp(A), ars, acs, _dp(B), brs, bcs, _dp(C), Nc, 1,
                     alg.M, alg.K, alg.N, alg.R, _dp(U), _dp(V), _dp(W), L)
    return C


def fast_entries(A: np.ndarray, B: np.ndarray, alg: Alg, L: int, rows, cols) -> np.ndarray:
    """Entries C[rows[e], cols[e]] of exactly fast(A, B, alg, L), computed one by one."""
    P, Q = A.shape
    _, Nc = B.shape
    U, V, W = _alg_arrays(alg)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(len(rows), dtype=np.float64)
    ars, acs = _strides(A); brs, bcs = _strides(B)
    p64 = ctypes.POINTER(ctypes.c_int64)
    _L().oracle_fast_entries(P, Q, Nc, _dp(A), ars, acs, _dp(B), brs, bcs,
                             alg.M, alg.K, alg.N, alg.R, _dp(U), _dp(V), _dp(W), L, len(rows),
                             rows.ctypes.data_as(p64), cols.ctypes.data_as(p64), _dp(out))
    return out


def classical_entries(A: np.ndarray, B: np.ndarray, rows, cols) -> np.ndarray:
    """Entries of the classical definition, one dot product each, q ascending (fast_entries
    with L = 0)."""
    return fast_entries(A, B, classical_alg(1, 1, 1), 0, rows, cols)


def flops(P: int, Q: int, Nc: int, alg: Alg, L: int) -> float:
    U, V, W = _alg_arrays(alg)
    return _L().oracle_flops(P, Q, Nc, alg.M, alg.K, alg.N, alg.R, _dp(U), _dp(V), _dp(W), L)


# --------------------------------------------------------------------------------------------
# addition-chain traffic per recursion node, in sub-block reads and writes (Sec. 3.2)
# --------------------------------------------------------------------------------------------
def addition_traffic(alg: Alg, strategy: str, alias_singletons: bool = False):
    """(reads, writes) of one recursion node's addition chains, counted chain by chain as the three
    implementations of P:622-636 perform them: the S_r chains (U columns), the T_r chains (V columns)
    and the C_k chains (W rows).
      pairwise   -- per chain of n terms: a copy (1 read, 1 write) then n - 1 daxpy calls (2 reads,
                    1 write each), P:622-626 and the footnote;
      write_once -- per chain: n reads, 1 write; U / V chains of one term are not written;
      streaming  -- every A, B and M_r block a chain uses is read once; every formed S_r, T_r
                    (more than one term) and every C_k is written once.
    alias_singletons: one-term U / V chains cost nothing at all, neither read nor write (the GPU
    path hands the block itself to the leaf product; SURVEY 8(d)'s "actual HBM traffic")."""
    U, V, W = alg.U, alg.V, alg.W
    R = alg.R
    ucols = [[i for i in range(len(U)) if U[i][r] != 0] for r in range(R)]
    vcols = [[j for j in range(len(V)) if V[j][r] != 0] for r in range(R)]
    wrows = [[r for r in range(R) if W[k][r] != 0] for k in range(len(W))]
    reads = writes = 0
    for side, chains in (("u", ucols), ("v", vcols), ("w", wrows)):
        if strategy == "streaming":
            used = set()
            for c in chains:
                if side != "w" and len(c) == 1 and alias_singletons:
                    continue
                used.update(c)
            reads += len(used)
        for c in chains:
            n = len(c)
            single = side != "w" and n == 1
            if single and alias_singletons:
                continue
            if strategy == "pairwise":
                reads += 2 * n - 1
                writes += n
            elif strategy == "write_once":
                reads += n
                writes += 0 if single else 1
            elif strategy == "streaming":
                writes += 0 if single else 1
            else:
                raise ValueError(strategy)
    return reads, writes


# --------------------------------------------------------------------------------------------
# check (d): a worst-case forward error bound derived from (U, V, W)
# --------------------------------------------------------------------------------------------
UNIT_ROUNDOFF = 2.0 ** -53


def _gamma(n: int) -> float:
    """gamma_n = n u / (1 - n u): the standard bound for n roundings in a sum or product chain."""
    nu = n * UNIT_ROUNDOFF
    return nu / (1.0 - nu)


def _chain_roundings(coefs) -> int:
    """Roundings of a chain sum_i c_i x_i evaluated term by term: one per addition, plus one per
    product c_i x_i whose coefficient is not a power of two (those products are exact)."""
    nz = [Fraction(c) for c in coefs if c != 0]
    def pow2(c):
        c = abs(c)
        return c.numerator & (c.numerator - 1) == 0 and c.denominator & (c.denominator - 1) == 0
    return max(0, len(nz) - 1) + sum(0 if pow2(c) else 1 for c in nz)


def error_bound(alg: Alg, Q: int, L: int, a: float = 1.0, b: float = 1.0) -> float:
    """Upper bound on max_ij |fl(C)_ij - (AB)_ij| for L recursive steps of `alg` (no peeling: Q a
    multiple of K^L) with ||A||_max <= a, ||B||_max <= b, any summation order inside each chain
    and a classical leaf of inner dimension Q / K^L (dot products with or without FMA).
    Recursion (max-norm, first order in the roundings but with exact gamma factors):
      leaf:  gamma_q q a b
      level: S_r = sum_i u_ir A_i  ->  |S_r| <= ||u_r||_1 a,  |fl(S_r) - S_r| <= gamma_{n_r} ||u_r||_1 a
             M_r = S_r T_r (recursively, on the rounded operands), plus the operand-error term
             q' (eS (|T| + eT) + |S| eT);   C_k = sum_r w_kr M_r rounded by gamma_{n_k}."""
    K = alg.K
    if L == 0:
        return _gamma(Q) * Q * a * b
    assert Q % K == 0, "error_bound covers unpeeled shapes"
    q = Q // K
    R = alg.R
    errM, magM = [], []
    for r in range(R):
        ucol = [alg.U[i][r] for i in range(alg.M * alg.K)]
        vcol = [alg.V[j][r] for j in range(alg.K * alg.N)]
        sa = float(sum(abs(Fraction(c)) for c in ucol)) * a
        tb = float(sum(abs(Fraction(c)) for c in vcol)) * b
        ea = _gamma(_chain_roundings(ucol)) * sa
        eb = _gamma(_chain_roundings(vcol)) * tb
        inner = error_bound(alg, q, L - 1, sa + ea, tb + eb)
        errM.append(inner + q * (ea * (tb + eb) + sa * eb))
        magM.append(q * sa * tb)
    worst = 0.0
    for k in range(alg.M * alg.N):
        wrow = [alg.W[k][r] for r in range(R)]
        absw = [float(abs(Fraction(c))) for c in wrow]
        e = sum(w * em for w, em in zip(absw, errM))
        e += _gamma(_chain_roundings(wrow)) * sum(w * (m + em) for w, m, em in zip(absw, magM, errM))
        worst = max(worst, e)
    return worst
