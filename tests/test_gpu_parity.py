"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances (BASELINE.json north star):
  max|C_gpu - C_oracle_fast| <= 1e-12 |A|_F |B|_F
  max|C_gpu - C_classical|   <= 1e-10 |A|_F |B|_F          (L <= 3)
Integer and quantised inputs make every rounding exact, so there the results must be bit-exact.
"""
import glob
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

NAMES = [os.path.basename(p)[:-4] for p in sorted(glob.glob(os.path.join(ALGS, "*.txt")))]
_ORA = {}


def oalg(name):
    if name not in _ORA:
        _ORA[name] = O.load_alg(os.path.join(ALGS, name + ".txt"))
    return _ORA[name]


_FA = {}


def falg(name):
    if name not in _FA:
        _FA[name] = F.load_alg(name)
    return _FA[name]


def dev(x, layout="row"):
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    if layout == "col":
        t = torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    return t


def run(name, A, B, L, layout="row", **kw):
    P, Q = A.shape
    N = B.shape[1]
    p = F.Plan(falg(name), P, Q, N, L, layout=layout, **kw)
    C = p.execute(dev(A, layout), dev(B, layout))
    torch.cuda.synchronize()
    return C.cpu().numpy(), p


def bound(A, B, c):
    return c * np.linalg.norm(A) * np.linalg.norm(B)


# ---- the DMMA GEMM kernel on its own ----------------------------------------------------------
@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (128, 128, 16), (256, 384, 512), (129, 257, 33), (300, 17, 1000),
                                   (7, 513, 64), (1000, 1000, 3)])
def test_dgemm_matches_classical(m, n, k):
    A, B = I.problem(m, k, n, seed=m + n + k)
    C = F.dgemm(dev(A), dev(B)).cpu().numpy()
    assert np.max(np.abs(C - O.classical(A, B))) <= bound(A, B, 1e-13)
    Ai, Bi = I.problem(m, k, n, seed=3, kind="integers")
    assert np.array_equal(F.dgemm(dev(Ai), dev(Bi)).cpu().numpy(), O.classical(Ai, Bi))


def test_dgemm_alpha_beta_and_unaligned_views():
    A, B = I.problem(200, 150, 170, seed=1, kind="integers")
    Cin = I.integers(9, 200, 170)
    # odd leading dimensions and odd offsets force the 8-byte copy path
    Abig = torch.zeros(201, 153, dtype=torch.float64, device="cuda")
    Abig[1:, 3:] = dev(A)
    Bbig = torch.zeros(151, 175, dtype=torch.float64, device="cuda")
    Bbig[1:, 5:] = dev(B)
    C = dev(Cin).clone()
    F.dgemm(Abig[1:, 3:], Bbig[1:, 5:], C, alpha=-2.0, beta=1.0)
    assert np.array_equal(C.cpu().numpy(), Cin - 2.0 * O.classical(A, B))


# ---- check (c) on the GPU: integer inputs are bit-exact ---------------------------------------
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("L", [1, 2])
def test_fast_integer_bit_exact(name, L):
    a = oalg(name)
    P, Q, N = 3 * a.M ** L + 1, 2 * a.K ** L + 1, 2 * a.N ** L + 2  # peeled at every level
    A, B = I.problem(P, Q, N, seed=L, kind="integers")
    C, _ = run(name, A, B, L)
    assert np.array_equal(C, O.classical(A, B))


def test_config1_4x4_integers():
    A, B = I.problem(4, 4, 4, seed=0, kind="integers")
    for L in (1, 2):
        C, _ = run("strassen_222_7", A, B, L)
        assert np.array_equal(C, A @ B)


# ---- float parity against oracle_fast at sizes spanning several tiles and a ragged tail -------
CASES = [
    ("strassen_222_7", 1, 256, 256, 256),                 # BASELINE config 1
    ("strassen_222_7", 3, 1000, 999, 1001),
    ("winograd_class_222_7", 2, 1024, 1024, 1024),
    ("winograd_class_222_7", 2, 777, 529, 901),
    ("hk_class_323_15", 2, 600, 90, 600),                  # config 3 shape family, peeled at level 2
    ("hk_class_323_15", 1, 451, 301, 452),
    ("alg_424_26", 2, 800, 120, 800),                      # config 4 family
    ("laderman_class_333_23", 2, 450, 450, 450),           # config 5 family
    ("laderman_class_333_23", 1, 331, 332, 333),
    ("alg_433_29", 2, 720, 144, 144),                      # config 5t family
    ("alg_433_29", 1, 401, 302, 299),
]


@pytest.mark.parametrize("name,L,P,Q,N", CASES)
@pytest.mark.parametrize("layout", ["row", "col"])
def test_fast_float_parity(name, L, P, Q, N, layout):
    A, B = I.problem(P, Q, N, seed=L + P)
    C, _ = run(name, A, B, L, layout=layout)
    ref = O.fast(A, B, oalg(name), L)
    assert np.max(np.abs(C - ref)) <= bound(A, B, 1e-12)
    assert np.max(np.abs(C - O.classical(A, B))) <= bound(A, B, 1e-10)


@pytest.mark.parametrize("strategy", ["streaming", "write_once", "pairwise"])
@pytest.mark.parametrize("cse", [False, True])
def test_strategies_and_cse(strategy, cse):
    for name, L, P, Q, N in [("alg_424_26", 2, 320, 64, 320), ("winograd_class_222_7", 2, 512, 512, 512)]:
        A, B = I.problem(P, Q, N, seed=5)
        C, _ = run(name, A, B, L, strategy=strategy, cse=cse)
        assert np.max(np.abs(C - O.fast(A, B, oalg(name), L))) <= bound(A, B, 1e-12)
        Ai, Bi = I.problem(P, Q, N, seed=6, kind="integers")
        Ci, _ = run(name, Ai, Bi, L, strategy=strategy, cse=cse)
        assert np.array_equal(Ci, Ai @ Bi)


@pytest.mark.parametrize("name,L,P,Q,N", [("strassen_222_7", 2, 256, 256, 256), ("alg_424_26", 2, 328, 66, 330),
                                           ("laderman_class_333_23", 1, 99, 96, 93)])
def test_three_strategies_round_identically(name, L, P, Q, N):
    # without CSE every strategy sums each chain in ascending index order: bitwise equal
    A, B = I.problem(P, Q, N, seed=12)
    # (the separate streaming kernels: the one-launch small path sums the leaf products' k in
    # another order)
    Cs, _ = run(name, A, B, L, strategy="streaming", cse=False, small=False)
    for strategy in ("write_once", "pairwise"):
        C, _ = run(name, A, B, L, strategy=strategy, cse=False)
        assert np.array_equal(C, Cs), strategy


def test_pairwise_traffic_is_the_papers_count():
    # pairwise reads 2 nnz(U,V,W) - 2R - MN and writes nnz(U,V,W) sub-blocks per node.
    # Strassen: nnz = 12 + 12 + 12, R = 7, MN = 4 -> 54 reads, 36 writes; the two singleton columns
    # of U and of V are aliased, not copied, which removes 4 reads and 4 writes.
    b = 256
    A, B = I.problem(2 * b, 2 * b, 2 * b, seed=13)
    C, p = run("strassen_222_7", A, B, 1, strategy="pairwise", cse=False)
    assert p.stats()["add_bytes"] == 8 * (50 + 32) * b * b
    # one launch per chain position: longest S chain 2, T chain 2, C chain 4, plus the leaf GEMM
    assert p.stats()["launches"] == 2 + 2 + 1 + 4
    assert np.max(np.abs(C - O.fast(A, B, oalg("strassen_222_7"), 1))) <= bound(A, B, 1e-12)
    _, pw = run("strassen_222_7", A, B, 1, strategy="write_once", cse=False)
    assert pw.stats()["add_bytes"] < p.stats()["add_bytes"]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("strategy", ["streaming", "write_once", "pairwise"])
def test_addition_bytes_equal_the_oracles_chain_count(name, strategy):
    # one level on b x b blocks: the plan's algorithmic addition bytes are the oracle's chain-by-chain
    # sub-block count (singleton chains aliased, as the kernels do) x 8 b^2
    a = falg(name)
    b = 64
    P, Q, N = a.M * b, a.K * b, a.N * b
    A, B = I.problem(P, Q, N, seed=14, kind="integers")
    C, p = run(name, A, B, 1, strategy=strategy, cse=False, small=False)  # the separate kernels' bytes
    reads, writes = O.addition_traffic(oalg(name), strategy, alias_singletons=True)
    assert p.stats()["add_bytes"] == 8 * b * b * (reads + writes)
    assert np.array_equal(C, A @ B)


def test_quantized_inputs_exact_at_scale():
    # g = 11 grid: every partial sum of classical and fast algorithms is exact
    for name, L, P, Q, N in [("winograd_class_222_7", 2, 2048, 2048, 2048), ("alg_433_29", 2, 1800, 360, 360)]:
        A, B = I.problem(P, Q, N, seed=7, kind="quantized")
        C, _ = run(name, A, B, L)
        s = 2.0 ** 11
        exact = ((A * s).astype(np.int64) @ (B * s).astype(np.int64)).astype(np.float64) / (s * s)
        assert np.array_equal(C, exact)


# ---- sharding (HYBRID arithmetic): shards sum to the product ----------------------
@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("mode", ["leaf", "top"])
def test_shards_sum_to_product(G, mode):
    for name, L, P, Q, N in [("winograd_class_222_7", 2, 300, 200, 250), ("hk_class_323_15", 2, 271, 181, 269),
                             ("alg_424_26", 2, 320, 64, 320)]:
        Ai, Bi = I.problem(P, Q, N, seed=8, kind="integers")
        total = np.zeros((P, N))
        for g in range(G):
            C, _ = run(name, Ai, Bi, L, shard_rank=g, shard_count=G, shard_mode=mode)
            total += C
        assert np.array_equal(total, Ai @ Bi)


def test_top_level_shards_more_ranks_than_products():
    # G > R: ranks beyond R own nothing and return zeros
    Ai, Bi = I.problem(96, 64, 80, seed=9, kind="integers")
    total = np.zeros((96, 80))
    for g in range(9):
        C, _ = run("strassen_222_7", Ai, Bi, 1, shard_rank=g, shard_count=9, shard_mode="top")
        if g >= 7:
            assert not C.any()
        total += C
    assert np.array_equal(total, Ai @ Bi)


# ---- edge cases -------------------------------------------------------------------------------
def test_degenerate_dims():
    a = falg("strassen_222_7")
    for (P, Q, N) in [(0, 5, 5), (5, 0, 5), (5, 5, 0), (1, 1, 1), (1, 7, 1), (3, 3, 3)]:
        A, B = I.problem(P, Q, N, seed=1, kind="integers")
        p = F.Plan(a, P, Q, N, 2)
        C = torch.full((P, N), 7.0, dtype=torch.float64, device="cuda")
        p.execute(dev(A) if A.size else torch.zeros(P, Q, dtype=torch.float64, device="cuda"),
                  dev(B) if B.size else torch.zeros(Q, N, dtype=torch.float64, device="cuda"), C)
        assert np.array_equal(C.cpu().numpy(), A @ B)


def test_levels_beyond_base_case_stop_early():
    A, B = I.problem(20, 20, 20, seed=2, kind="integers")
    C, p = run("laderman_class_333_23", A, B, 8)
    assert np.array_equal(C, A @ B)
    assert p.stats()["levels"] == 2  # 20 -> 6 -> 2 < 3


def test_strided_inputs_and_output():
    A, B = I.problem(130, 66, 98, seed=4)
    Ab = torch.zeros(130, 80, dtype=torch.float64, device="cuda"); Ab[:, :66] = dev(A)
    Bb = torch.zeros(66, 111, dtype=torch.float64, device="cuda"); Bb[:, 5:103] = dev(B)
    Cb = torch.zeros(130, 200, dtype=torch.float64, device="cuda")
    p = F.Plan(falg("strassen_222_7"), 130, 66, 98, 2)
    p.execute(Ab[:, :66], Bb[:, 5:103], Cb[:, 1:99])
    ref = O.fast(A, B, oalg("strassen_222_7"), 2)
    assert np.max(np.abs(Cb[:, 1:99].cpu().numpy() - ref)) <= bound(A, B, 1e-12)
    assert not Cb[:, 0].any() and not Cb[:, 99:].any()  # nothing written outside C


def test_deterministic():
    A, B = I.problem(513, 257, 515, seed=9)
    p = F.Plan(falg("alg_424_26"), 513, 257, 515, 2)
    C1 = p.execute(dev(A), dev(B)).clone()
    C2 = p.execute(dev(A), dev(B))
    assert torch.equal(C1, C2)


def test_errors_are_reported():
    p = F.Plan(falg("strassen_222_7"), 8, 8, 8, 1)
    with pytest.raises(ValueError):
        p.execute(torch.zeros(8, 9, dtype=torch.float64, device="cuda"), torch.zeros(8, 8, dtype=torch.float64, device="cuda"))
    with pytest.raises(F.FmmError) as e:
        F.Plan(falg("strassen_222_7"), -1, 8, 8, 1)
    assert e.value.status == "FMM_E_SHAPE"


@pytest.mark.parametrize("layout", ["row", "col"])
def test_tile_aware_row_peel(layout):
    # R7c: leaves of 130 rows would take two 128-row tiles; with peel_tiles the plan peels 2 rows of
    # every leaf into the classical strips (the cost model prefers it here) -- still exact
    P, Q, N = 9 * 130, 4 * 64, 9 * 130
    A, B = I.problem(P, Q, N, seed=15, kind="integers")
    C, p = run("hk_class_323_15", A, B, 2, layout=layout, peel_tiles=True)
    assert p.stats()["tiled_peel"] == 1 and np.array_equal(C, A @ B)
    C, p = run("hk_class_323_15", A, B, 2, layout=layout)
    assert p.stats()["tiled_peel"] == 0 and np.array_equal(C, A @ B)


def test_option_errors_are_reported():
    # the workspace limit (the message states the R-fold requirement)
    with pytest.raises(F.FmmError) as e:
        F.Plan(falg("strassen_222_7"), 512, 512, 512, 2, workspace_limit_bytes=1 << 20)
    assert e.value.status == "FMM_E_NO_MEMORY" and "workspace bytes" in str(e.value)
    F.Plan(falg("strassen_222_7"), 512, 512, 512, 2, workspace_limit_bytes=1 << 30)  # fits
    with pytest.raises(F.FmmError) as e:
        F.Plan(falg("strassen_222_7"), 64, 64, 64, 1, shard_rank=3, shard_count=2)
    assert e.value.status == "FMM_E_INVALID_ARG"
    with pytest.raises(ValueError):
        F.Plan(falg("strassen_222_7"), 64, 64, 64, 1, strategy="daxpy")
    comm = F.Comm(F.nccl_unique_id(), 1, 0)
    with pytest.raises(F.FmmError) as e:
        F.Plan(falg("strassen_222_7"), 64, 64, 64, 1, comm=comm, root=1)
    assert e.value.status == "FMM_E_INVALID_ARG"
    # C overlapping A or B is refused before any device work
    p = F.Plan(falg("strassen_222_7"), 64, 64, 64, 1)
    X = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    Y = torch.zeros(64, 64, dtype=torch.float64, device="cuda")
    for args in [(X, Y, X), (X, Y, Y)]:
        with pytest.raises(F.FmmError) as e:
            p.execute(*args)
        assert e.value.status == "FMM_E_INVALID_ARG"
    big = torch.zeros(128, 64, dtype=torch.float64, device="cuda")
    p.execute(big[:64], Y, big[64:])  # adjacent, not overlapping: fine


def test_execute_host_end_to_end():
    A, B = I.problem(300, 200, 310, seed=10)
    p = F.Plan(falg("hk_class_323_15"), 300, 200, 310, 2)
    C = np.zeros((300, 310))
    p.execute_host(A, B, C)
    assert np.max(np.abs(C - O.fast(A, B, oalg("hk_class_323_15"), 2))) <= bound(A, B, 1e-12)


def test_cp_async_gemm_path_matches_tma_path(monkeypatch):
    # FMM_NO_TMA=1 forces the cp.async grouped GEMM; both must give oracle parity
    A, B = I.problem(700, 300, 650, seed=11)
    ref = O.fast(A, B, oalg("alg_424_26"), 2)
    C_tma, _ = run("alg_424_26", A, B, 2)
    monkeypatch.setenv("FMM_NO_TMA", "1")
    C_cp, _ = run("alg_424_26", A, B, 2)
    for C in (C_tma, C_cp):
        assert np.max(np.abs(C - ref)) <= bound(A, B, 1e-12)


@pytest.mark.parametrize("peel_align", [False, True])
def test_peel_modes_and_thin_strips(peel_align):
    # c3's shape family at small scale: odd level-2 column blocks (paper peeling) vs aligned peeling;
    # both give oracle parity, and integer inputs stay bit-exact (thin strips run on CUDA cores)
    for name, L, P, Q, N in [("hk_class_323_15", 2, 400, 60, 400), ("strassen_222_7", 2, 203, 101, 207)]:
        A, B = I.problem(P, Q, N, seed=12)
        C, _ = run(name, A, B, L, peel_align=peel_align)
        assert np.max(np.abs(C - O.fast(A, B, oalg(name), L))) <= bound(A, B, 1e-12)
        Ai, Bi = I.problem(P, Q, N, seed=13, kind="integers")
        Ci, _ = run(name, Ai, Bi, L, peel_align=peel_align)
        assert np.array_equal(Ci, Ai @ Bi)


@pytest.mark.parametrize("bn", ["128", "112", "96", "80", "64"])
def test_every_tma_tile_width(bn, monkeypatch):
    monkeypatch.setenv("FMM_GEMM_BN", bn)
    A, B = I.problem(300, 200, 333, seed=14)
    ref = O.classical(A, B)
    C = F.dgemm(dev(A), dev(B)).cpu().numpy()
    assert np.max(np.abs(C - ref)) <= bound(A, B, 1e-13)
    Ai, Bi = I.problem(260, 72, 410, seed=15, kind="integers")
    C, _ = run("alg_433_29", Ai, Bi, 1)
    assert np.array_equal(C, Ai @ Bi)


@pytest.mark.parametrize("epi", ["1", "2"])
@pytest.mark.parametrize("bn", ["128", "112", "80", "64"])
def test_staged_epilogue(epi, bn, monkeypatch):
    # the leaf GEMM's staged bulk-copy epilogue (FMM_GEMM_EPI, DESIGN 6d): ragged rows, an odd
    # column count (the last column stored directly), several tiles per CTA (slot hand-over)
    monkeypatch.setenv("FMM_GEMM_EPI", epi)
    monkeypatch.setenv("FMM_GEMM_BN", bn)
    A, B = I.problem(300, 200, 333, seed=16)
    C = F.dgemm(dev(A), dev(B)).cpu().numpy()
    assert np.max(np.abs(C - O.classical(A, B))) <= bound(A, B, 1e-13)
    Ai, Bi = I.problem(1037, 96, 1201, seed=17, kind="integers")
    C, _ = run("alg_433_29", Ai, Bi, 1)
    assert np.array_equal(C, Ai @ Bi)
    A, B = I.problem(2050, 300, 1999, seed=18)
    C, _ = run("winograd_class_222_7", A, B, 2)
    assert np.max(np.abs(C - O.fast(A, B, oalg("winograd_class_222_7"), 2))) <= bound(A, B, 1e-12)


def test_execute_host_async_pipeline():
    # three back-to-back pipelined host calls with different inputs and outputs
    import torch as T
    name, L, P, Q, N = "winograd_class_222_7", 2, 256, 192, 320
    p = F.Plan(falg(name), P, Q, N, L)
    outs, refs = [], []
    for s in range(3):
        A, B = I.problem(P, Q, N, seed=20 + s)
        Ah, Bh = T.from_numpy(A).pin_memory(), T.from_numpy(B).pin_memory()
        Ch = T.zeros(P, N, dtype=T.float64).pin_memory()
        p.execute_host(Ah, Bh, Ch, asynchronous=True)
        outs.append((Ah, Bh, Ch))
        refs.append(O.fast(A, B, oalg(name), L))
    p.sync()
    for (Ah, Bh, Ch), ref in zip(outs, refs):
        assert np.max(np.abs(Ch.numpy() - ref)) <= bound(Ah.numpy(), Bh.numpy(), 1e-12)


# ---- check (d) on the GPU: the error stays within the bound derived from (U, V, W) -------------
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("L", [1, 2])
@pytest.mark.parametrize("layout", ["row", "col"])
def test_gpu_error_within_derived_bound(name, L, layout):
    a = oalg(name)
    P, Q, N = a.M ** L * 40, a.K ** L * 48, a.N ** L * 36
    A, B = I.problem(P, Q, N, seed=40 + L)
    C, _ = run(name, A, B, L, layout=layout)
    exact = A.astype(np.longdouble) @ B.astype(np.longdouble)
    err = float(np.max(np.abs(C.astype(np.longdouble) - exact)))
    assert err <= O.error_bound(a, Q, L, float(np.abs(A).max()), float(np.abs(B).max()))


# ---- the library's own multi-GPU combine (fmm_comm_create / fmm_plan_create_dist) -------------
def test_distributed_plan_single_rank():
    # one rank: the NCCL reduce to the root is a no-op copy, so the distributed plan must equal the
    # local one; a non-contiguous C is refused
    A, B = I.problem(300, 200, 250, seed=21, kind="integers")
    comm = F.Comm(F.nccl_unique_id(), 1, 0)
    p = F.Plan(falg("winograd_class_222_7"), 300, 200, 250, 2, comm=comm, root=0)
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), A @ B)
    Cb = torch.zeros(300, 260, dtype=torch.float64, device="cuda")
    with pytest.raises(F.FmmError) as e:
        p.execute(dev(A), dev(B), Cb[:, :250])
    assert e.value.status == "FMM_E_UNSUPPORTED"


@pytest.mark.parametrize("layout", ["row", "col"])
def test_distributed_plan_single_rank_slabs(layout):
    # root = "slabs" (FMM_DIST_SLABS) at one rank: the only slab is all of C
    A, B = I.problem(260, 130, 190, seed=22, kind="integers")
    comm = F.Comm(F.nccl_unique_id(), 1, 0)
    p = F.Plan(falg("alg_424_26"), 260, 130, 190, 2, layout=layout, comm=comm, root="slabs")
    C = p.execute(dev(A, layout), dev(B, layout))
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), A @ B)
    assert F.dist_slab(260, 190, layout, 1, 0) == (0, 260 if layout == "row" else 190)


def test_classical_root_shards_write_zeros_elsewhere():
    # L = 0 (or a problem below the base case): the root is the only leaf and its rows are split
    # across shards; every shard must write zeros in the rows it does not own (found by
    # tests/test_gpu_random.py: a 1 x 1 x 1 problem over 2 shards summed uninitialised memory)
    for (P, Q, N, L) in [(1, 1, 1, 2), (5, 3, 4, 0), (300, 64, 70, 0)]:
        A, B = I.problem(P, Q, N, seed=P, kind="integers")
        for G in (2, 3):
            total = np.zeros((P, N))
            for g in range(G):
                p = F.Plan(falg("alg_424_26"), P, Q, N, L, shard_rank=g, shard_count=G)
                C = torch.full((P, N), float("nan"), dtype=torch.float64, device="cuda")
                p.execute(dev(A), dev(B), C)
                torch.cuda.synchronize()
                total += C.cpu().numpy()
            assert np.array_equal(total, A @ B)


@pytest.mark.parametrize("alg,shape,layout,chunks,root", [
    ("winograd_class_222_7", (256, 256, 256), "col", 4, 0),       # collapsed two-level assembly writes C
    ("winograd_class_222_7", (301, 200, 250), "row", 3, 0),       # bottom peel rows: the tail reduce
    ("hk_class_323_15", (301, 64, 299), "row", 7, "slabs"),       # top-level row and column strips
    ("alg_424_26", (257, 131, 190), "col", 4, 0),                 # K peel at the top: one reduce at the end
    ("alg_433_29", (180, 36, 36), "row", 1, 0)])                  # chunking off
def test_distributed_plan_chunked_reduce(alg, shape, layout, chunks, root):
    # NCCL plan, dist_chunks row chunks of the C-writing assembly, each reduced on the library's comm
    # stream; at one rank every reduce is an in-place copy, so C must be the exact product whatever
    # the chunking (it checks the chunk tables, the strip reordering and the tail rows)
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=23, kind="integers")
    comm = F.Comm(F.nccl_unique_id(), 1, 0)
    p = F.Plan(falg(alg), P, Q, N, 2, layout=layout, comm=comm, root=root, dist_chunks=chunks)
    for _ in range(2):
        C = p.execute(dev(A, layout), dev(B, layout))
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), A @ B)
    _, t = p.execute_timed(dev(A, layout), dev(B, layout), C)
    assert t["gemm_ms"] > 0 and t["total_ms"] >= t["gemm_ms"]


@pytest.mark.parametrize("alg,shape,layout,mode,G", [("alg_424_26", (640, 200, 640), "row", "top", 3),
                                                     ("hk_class_323_15", (361, 120, 363), "col", "top", 4),
                                                     ("winograd_class_222_7", (256, 256, 256), "row", "leaf", 4),
                                                     ("alg_433_29", (480, 96, 96), "row", "leaf", 8)])
def test_shard_reads_only_its_input_blocks(alg, shape, layout, mode, G):
    # fmm_plan_input_blocks: a shard reads only the top-level A / B blocks its level-1 products touch
    # (send a rank only those).  Poison every other block -- and the peeled edges unless
    # the shard owns the top-level strips -- with NaN: the shard's partial product must not change.
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=24, kind="integers")
    a = falg(alg)
    restricted = 0
    for g in range(G):
        p = F.Plan(a, P, Q, N, 2, layout=layout, shard_rank=g, shard_count=G, shard_mode=mode)
        needA, needB, (P1, Q1, N1), need_all = p.input_blocks()
        clean = p.execute(dev(A, layout), dev(B, layout)).cpu().numpy()
        if need_all:
            continue
        Ap, Bp = A.copy(), B.copy()
        pb, qb, nb = P1 // a.M, Q1 // a.K, N1 // a.N
        keepA = np.zeros_like(A, dtype=bool)
        keepB = np.zeros_like(B, dtype=bool)
        for i, need in enumerate(needA):
            if need:
                x, y = divmod(i, a.K)
                keepA[x * pb:(x + 1) * pb, y * qb:(y + 1) * qb] = True
        for j, need in enumerate(needB):
            if need:
                x, y = divmod(j, a.N)
                keepB[x * qb:(x + 1) * qb, y * nb:(y + 1) * nb] = True
        Ap[~keepA] = np.nan
        Bp[~keepB] = np.nan
        restricted += int(not (keepA.all() and keepB.all()))
        got = p.execute(dev(Ap, layout), dev(Bp, layout)).cpu().numpy()
        assert np.array_equal(got, clean), (g, np.isnan(got).sum())
    print(f"{alg} {mode} G={G}: {restricted} of {G} shards read a strict subset of A and B")
    assert restricted >= 1  # measured: 2 of 3, 3 of 4, 2 of 4, 8 of 8 for the four cases


@pytest.mark.parametrize("alg,shape,layout,L", [("winograd_class_222_7", (512, 512, 512), "col", 2),
                                                ("hk_class_323_15", (301, 200, 299), "row", 2)])
def test_execute_profile_lists_every_launch(alg, shape, layout, L):
    # fmm_execute_profile: one entry per launch of the step (kind, recursion level, time); the kinds
    # follow the plan's structure and the launch count matches fmm_plan_stats
    P, Q, N = shape
    A, B = I.problem(P, Q, N, seed=25, kind="integers")
    p = F.Plan(falg(alg), P, Q, N, L, layout=layout)
    C = p.new_output()
    p.execute(dev(A, layout), dev(B, layout), C)  # first use: module loading, kernel attributes
    prof = p.execute_profile(dev(A, layout), dev(B, layout), C)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), A @ B)
    kinds = [k for k, _, _ in prof]
    assert kinds.count("leaf_gemm") == 1 and all(ms >= 0 for _, _, ms in prof)
    assert kinds.index("form_A") < kinds.index("leaf_gemm") < kinds.index("assembly")
    st = p.stats()
    assert len(prof) <= st["launches"]  # a thin-strip entry can hold two kernel launches
    _, t = p.execute_timed(dev(A, layout), dev(B, layout), C)
    assert abs(sum(ms for _, _, ms in prof) - t["total_ms"]) < 0.5 * t["total_ms"] + 0.05


# ---- thin peel strips: both row-strip forms (fmm_skinny.cu) --------------------
# Strip heights 1-7 (TH 1, 2, 4, 8), k below / at / above the pipelined batch (4 slices x 4 rows,
# two batches in flight), ragged and odd column counts (the 128-column block's tail, a lone last
# column), row- and column-major; integer inputs, so every case is bit-exact against int64 matmul.
_STRIP_CASES = [("alg_433_29", 1, 4 * 37 + 3, 3 * 5 + 2, 3 * 43 + 2),
                ("alg_433_29", 1, 4 * 40 + 1, 3 * 11, 3 * 90 + 1),
                ("hk_class_323_15", 2, 9 * 31 + 5, 4 * 9 + 3, 9 * 29 + 7),
                ("hk_class_323_15", 1, 3 * 70 + 2, 2 * 1 + 1, 3 * 45 + 1),
                ("strassen_222_7", 2, 4 * 50 + 3, 4 * 40 + 1, 4 * 64 + 3),
                ("alg_424_26", 1, 4 * 30 + 3, 2 * 17 + 1, 4 * 33 + 3)]


def _strip_cases_check():
    for name, L, P, Q, N in _STRIP_CASES:
        for layout in ("row", "col"):
            Ai, Bi = I.problem(P, Q, N, seed=P + Q + N, kind="integers")
            C, p = run(name, Ai, Bi, L, layout=layout, peel_align=False)
            assert np.array_equal(C, Ai @ Bi), (name, L, P, Q, N, layout)


def test_thin_strips_row_forms():
    assert "alg_424_26" in NAMES
    _strip_cases_check()  # the default (wide) row-strip form


def test_thin_strips_row_forms_narrow():
    # the 32-column row-strip form, selected once per process by FMM_SKINNY_ROWS=narrow
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = ("import sys; sys.path[:0] = [%r, %r]; import test_gpu_parity as T; T._strip_cases_check(); print('ok')"
            % (here, os.path.dirname(here)))
    env = dict(os.environ, FMM_SKINNY_ROWS="narrow")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
