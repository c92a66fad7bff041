"""Seeded synthetic inputs shared by the oracle side and the CUDA side (tests, bench, smoke).

This module holds NO arithmetic of the method: it only draws matrices.  Reading R13 of DESIGN.md:
A and B are uniform[-1,1) fp64 from numpy's PCG64 with seeds s and s+1, filled as the logical
(row, col) matrix; a column-major run stores the same logical matrix in Fortran order.  Test-only
variants: small integers in [-3,3] (BASELINE config 1) and uniform values quantised to a 2^-g
grid (g = 11) so every product and partial sum of both the classical and the fast algorithms is
exact in fp64 ("exactness trick").
"""
import numpy as np


def _gen(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform(seed: int, rows: int, cols: int) -> np.ndarray:
    return _gen(seed).uniform(-1.0, 1.0, size=(rows, cols))


def integers(seed: int, rows: int, cols: int, lo: int = -3, hi: int = 3) -> np.ndarray:
    return _gen(seed).integers(lo, hi + 1, size=(rows, cols)).astype(np.float64)


def quantized(seed: int, rows: int, cols: int, g: int = 11) -> np.ndarray:
    scale = float(2 ** g)
    return np.round(_gen(seed).uniform(-1.0, 1.0, size=(rows, cols)) * scale) / scale


def problem(P: int, Q: int, Nc: int, seed: int = 0, kind: str = "uniform", layout: str = "row"):
    """(A, B) for C = A*B with A P x Q (seed), B Q x Nc (seed+1)."""
    f = {"uniform": uniform, "integers": integers, "quantized": quantized}[kind]
    A = f(seed, P, Q)
    B = f(seed + 1, Q, Nc)
    if layout == "col":
        A, B = np.asfortranarray(A), np.asfortranarray(B)
    return A, B


def sample_indices(seed: int, P: int, Nc: int, count: int):
    """Sampled output positions, always including the four corners and the last row/column
    (where peeling strips live)."""
    g = _gen(seed + 12345)
    r = list(g.integers(0, P, size=count))
    c = list(g.integers(0, Nc, size=count))
    r += [0, 0, P - 1, P - 1, P // 2, P - 1]
    c += [0, Nc - 1, 0, Nc - 1, Nc - 1, Nc // 2]
    return np.array(r, dtype=np.int64), np.array(c, dtype=np.int64)
