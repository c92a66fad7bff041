"""The fused leaf-level launch: level-L formation, the leaf DMMA GEMM and the level-L assembly in
one cooperative kernel -- fuse_leaf_level = 1 with addition CTAs on their own SMs, 2 with the jobs in
the GEMM CTAs' spare producer warps (background mode).

CPU: the NVRTC-generated fused kernel compiles for every algorithm, layout and tile width.
GPU: it evaluates the same generated chains as the separate K1/K3 kernels, so fused == separate
bitwise (with and without CSE); against the oracle it meets the north-star tolerance; integer
inputs stay bit-exact; leaf shards still sum to the product; every addition-CTA count works.
"""
import glob
import os

import numpy as np
import pytest

import fmm_inputs as I
from conftest import ALGS
from oracle import oracle as O

NAMES = [os.path.basename(p)[:-4] for p in sorted(glob.glob(os.path.join(ALGS, "*.txt")))]


def _lib():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


@pytest.mark.parametrize("name,layout,cse,bn", [("strassen_222_7", "row", True, 128), ("winograd_class_222_7", "col", True, 96),
                                              ("hk_class_323_15", "row", False, 112), ("alg_433_29", "row", True, 80),
                                              ("alg_424_26", "col", False, 64)])
def test_fused_kernel_compiles(name, layout, cse, bn):
    # host-only NVRTC compile (a few seconds each); the GPU tests below cover every algorithm
    F = _lib()
    F.fmm.fused_compile_check(F.load_alg(name), layout=layout, cse=cse, bn=bn)


@pytest.mark.parametrize("name,layout,bn,ks", [("winograd_class_222_7", "col", 128, 48), ("alg_424_26", "row", 112, 32),
                                               ("alg_433_29", "row", 128, 16)])
def test_fused_background_kernel_compiles(name, layout, bn, ks):
    F = _lib()
    F.fmm.fused_compile_check(F.load_alg(name), layout=layout, cse=True, bn=bn, ks=ks, mode=2)
    with pytest.raises(F.FmmError):
        F.fmm.fused_compile_check(F.load_alg(name), layout=layout, cse=True, bn=bn, ks=24, mode=2)


# ---- GPU ----------------------------------------------------------------------------------------
CASES = [
    ("strassen_222_7", 1, 256, 256, 256, "row"),
    ("strassen_222_7", 2, 512, 384, 640, "row"),
    ("winograd_class_222_7", 2, 1024, 1024, 1024, "col"),
    ("winograd_class_222_7", 2, 777, 529, 901, "row"),      # ragged: peeled at both levels
    ("hk_class_323_15", 2, 1203, 602, 1205, "row"),
    ("alg_424_26", 2, 1600, 240, 1600, "row"),
    ("alg_433_29", 2, 1800, 360, 360, "row"),
    ("laderman_class_333_23", 2, 900, 900, 900, "row"),
    ("laderman_class_333_23", 1, 331, 332, 333, "col"),
]


def _run(F, name, A, B, L, layout="row", **kw):
    import torch
    P, Q = A.shape
    N = B.shape[1]

    def dev(x):
        if layout == "row":
            return torch.from_numpy(np.ascontiguousarray(x)).cuda()
        return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    kw.setdefault("collapse", False)  # collapsed levels take precedence over the fused leaf level
    kw.setdefault("small", False)  # compare against the separate launches, not the one-launch small path
    p = F.Plan(F.load_alg(name), P, Q, N, L, layout=layout, **kw)
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy(), p.stats()


@pytest.mark.gpu
@pytest.mark.parametrize("name,L,P,Q,N,layout", CASES)
@pytest.mark.parametrize("cse", [False, True])
@pytest.mark.parametrize("mode", [1, 2])
def test_fused_equals_separate_and_oracle(name, L, P, Q, N, layout, cse, mode):
    F = _lib()
    A, B = I.problem(P, Q, N, seed=3 + P)
    Cf, sf = _run(F, name, A, B, L, layout, cse=cse, fuse=mode)
    Cs, ss = _run(F, name, A, B, L, layout, cse=cse, fuse=False)
    assert ss["fused_launches"] == 0
    if sf["fused_launches"]:
        assert sf["launches"] < ss["launches"]
    assert np.array_equal(Cf, Cs)  # the same generated chains, the same leaf GEMM
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    assert np.max(np.abs(Cf - O.fast(A, B, O.load_alg(F.alg_path(name)), L))) <= 1e-12 * nrm
    assert np.max(np.abs(Cf - O.classical(A, B))) <= 1e-10 * nrm


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [1, 2])
def test_fused_is_used_where_eligible(mode):
    F = _lib()
    A, B = I.problem(1024, 1024, 1024, seed=1)
    _, st = _run(F, "winograd_class_222_7", A, B, 2, fuse=mode)
    assert st["fused_launches"] == 1 and st["fused_add_bytes"] > 0


@pytest.mark.gpu
def test_fused_background_wins_over_collapse():
    # fuse_leaf_level = 2 takes precedence over collapse_levels (mode 1 yields to it)
    F = _lib()
    A, B = I.problem(1024, 1024, 1024, seed=1)
    _, s1 = _run(F, "winograd_class_222_7", A, B, 2, fuse=1, collapse=True)
    _, s2 = _run(F, "winograd_class_222_7", A, B, 2, fuse=2, collapse=True)
    assert s1["fused_launches"] == 0 and s1["collapsed"] == 1
    assert s2["fused_launches"] == 1 and s2["collapsed"] == 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("mode", [1, 2])
def test_fused_integer_bit_exact(name, mode):
    F = _lib()
    a = O.load_alg(F.alg_path(name))
    P, Q, N = 3 * a.M ** 2 + 1, 2 * a.K ** 2 + 1, 2 * a.N ** 2 + 2
    A, B = I.problem(P, Q, N, seed=2, kind="integers")
    C, _ = _run(F, name, A, B, 2, fuse=mode)
    assert np.array_equal(C, A @ B)


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("mode", [1, 2])
def test_fused_shards_sum_to_product(G, mode):
    F = _lib()
    A, B = I.problem(300, 200, 250, seed=8, kind="integers")
    total = np.zeros((300, 250))
    for g in range(G):
        C, _ = _run(F, "winograd_class_222_7", A, B, 2, fuse=mode, shard_rank=g, shard_count=G)
        total += C
    assert np.array_equal(total, A @ B)


@pytest.mark.gpu
@pytest.mark.parametrize("k", ["1", "7", "74", "147"])
def test_fused_any_addition_cta_count(k, monkeypatch):
    # from one addition CTA to one GEMM CTA: the dependency protocol must not deadlock
    F = _lib()
    monkeypatch.setenv("FMM_FUSE_ADD_CTAS", k)
    A, B = I.problem(640, 256, 512, seed=4, kind="integers")
    C, _ = _run(F, "alg_424_26", A, B, 2, fuse=True)
    assert np.array_equal(C, A @ B)
