"""GPU parity of the one-launch path for small one-level plans (option small_fused, DESIGN.md
sec. 6h) against the CPU oracle: every algorithm file bit-exact on integer inputs, ragged leaf
tiles, uniform inputs at the north-star tolerance, the c1 workload, and the option / cutoff rules."""
import os

import numpy as np
import pytest

import fmm_inputs as I
from conftest import ALGS
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_1409_2908_b200 as F

NAMES = sorted(os.path.basename(p)[:-4] for p in os.listdir(ALGS) if p.endswith(".txt"))


def plan(name, P, Q, N, L=1, **kw):
    return F.Plan(F.load_alg(name), P, Q, N, L, **kw)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("variant", ["coop", "last", "cluster"])
@pytest.mark.parametrize("name", NAMES)
def test_every_algorithm_exact(name, variant, monkeypatch):
    # the three assemblies: the R CTAs of a tile together (the grid is resident), the last CTA of
    # each tile, and the cluster variant where R <= 16 (C_k over distributed shared memory)
    monkeypatch.setenv("FMM_SMALL_CLUSTER", "1" if variant == "cluster" else "0")
    monkeypatch.setenv("FMM_SMALL_COOP", "1" if variant == "coop" else "0")
    alg = O.load_alg(os.path.join(ALGS, name + ".txt"))
    M, K, N = alg.M, alg.K, alg.N
    # leaves of 37 x 70 x 46: ragged 32 x 32 tiles, two k chunks of 64 (the second ragged)
    P, Q, Nc = 37 * M, 70 * K, 46 * N
    A, B = I.problem(P, Q, Nc, seed=3, kind="integers")
    p = plan(name, P, Q, Nc)
    assert p.stats()["small_fused"] == 1.0
    assert p.stats()["launches"] == 1.0
    C = p.execute(dev(A), dev(B))
    C2 = p.execute(dev(A), dev(B))  # the counters reset themselves between launches
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), A @ B)
    assert np.array_equal(C2.cpu().numpy(), A @ B)


@pytest.mark.parametrize("variant", ["coop", "last", "cluster"])
@pytest.mark.parametrize("shape", [(256, 256, 256), (2, 2, 2), (66, 130, 98), (500, 8, 300), (64, 2000, 64),
                                   (1024, 64, 1024)])
def test_uniform_against_oracle(shape, variant, monkeypatch):
    monkeypatch.setenv("FMM_SMALL_CLUSTER", "1" if variant == "cluster" else "0")
    monkeypatch.setenv("FMM_SMALL_COOP", "1" if variant == "coop" else "0")
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=P + Q + N)
    name = "strassen_222_7"
    p = plan(name, P, Q, N)
    assert p.stats()["small_fused"] == 1.0
    C = p.execute(dev(A), dev(B)).cpu().numpy()
    ref = O.fast(A, B, O.load_alg(os.path.join(ALGS, name + ".txt")), 1)
    tol = 1e-12 * np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(C - ref)) <= tol
    assert np.max(np.abs(C - O.classical(A, B))) <= 1e-10 * np.linalg.norm(A) * np.linalg.norm(B)


def test_column_major_and_leading_dimensions():
    P, Q, N = 200, 96, 144
    A, B = I.problem(P, Q, N, seed=9, kind="integers")
    p = plan("winograd_class_222_7", P, Q, N, layout="col")
    assert p.stats()["small_fused"] == 1.0
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda().t()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().t()
    C = p.execute(Ad, Bd)
    assert np.array_equal(C.cpu().numpy(), A @ B)
    # row-major views with padded leading dimensions
    Ab = torch.zeros(P, Q + 6, dtype=torch.float64, device="cuda")
    Bb = torch.zeros(Q, N + 10, dtype=torch.float64, device="cuda")
    Cb = torch.full((P, N + 2), 7.0, dtype=torch.float64, device="cuda")
    Ab[:, :Q] = dev(A)
    Bb[:, :N] = dev(B)
    q = plan("winograd_class_222_7", P, Q, N)
    q.execute(Ab[:, :Q], Bb[:, :N], Cb[:, :N])
    assert np.array_equal(Cb[:, :N].cpu().numpy(), A @ B)
    assert bool((Cb[:, N:] == 7.0).all())


def test_same_result_as_separate_launches():
    P, Q, N = 256, 256, 256
    A, B = I.problem(P, Q, N, seed=1)
    a = plan("strassen_222_7", P, Q, N)
    b = plan("strassen_222_7", P, Q, N, small=False)
    assert a.stats()["small_fused"] == 1.0 and b.stats()["small_fused"] == 0.0
    assert b.stats()["launches"] == 4.0
    Ca = a.execute(dev(A), dev(B)).cpu().numpy()
    Cb = b.execute(dev(A), dev(B)).cpu().numpy()
    assert np.max(np.abs(Ca - Cb)) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(B)


def test_not_applied_where_it_does_not_fit():
    # two levels, a peeled top level, or leaf products that fill the GPU keep the separate launches
    assert plan("strassen_222_7", 256, 256, 256, L=2).stats()["small_fused"] == 0.0
    assert plan("strassen_222_7", 257, 256, 256).stats()["small_fused"] == 0.0
    assert plan("strassen_222_7", 4096, 512, 4096).stats()["small_fused"] == 0.0
    assert plan("strassen_222_7", 256, 256, 256, fuse_output=True).stats()["small_fused"] == 0.0


@pytest.mark.parametrize("shape", [(256, 256, 256), (1, 1, 1), (100, 37, 250), (512, 1024, 300)])
def test_classical_below_the_cutoff(shape):
    # L = 0 below the cutoff: the classical product through the same one launch (base case
    # <1,1,1;1>, each CTA writes its tile of C directly)
    P, Q, N = shape
    p = plan("strassen_222_7", P, Q, N, L=0)
    assert p.stats()["small_fused"] == 1.0 and p.stats()["launches"] == 1.0
    A, B = I.problem(P, Q, N, seed=P + 2 * Q + 3 * N)
    C = p.execute(dev(A), dev(B)).cpu().numpy()
    assert np.max(np.abs(C - O.classical(A, B))) <= 1e-13 * np.linalg.norm(A) * np.linalg.norm(B)
    Ai, Bi = I.problem(P, Q, N, seed=5, kind="integers")
    assert np.array_equal(p.execute(dev(Ai), dev(Bi)).cpu().numpy(), Ai @ Bi)
    # large products keep the grouped GEMM
    assert plan("strassen_222_7", 4096, 256, 4096, L=0).stats()["small_fused"] == 0.0
