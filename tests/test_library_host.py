"""Host-side checks of the C-ABI library (no GPU): it loads, exports every symbol include/fmm.h
declares, and its host logic (exact Brent validation, file parser, HYBRID split arithmetic)
behaves as the paper fixes.  No compute call is made here."""
import ctypes
import glob
import os
import re
import subprocess

import pytest

from conftest import ALGS, GOLDEN, ROOT
from oracle import oracle as O

HEADER = os.path.join(ROOT, "include", "fmm.h")


@pytest.fixture(scope="module")
def F():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(F):
    names = declared_functions()
    assert len(names) >= 15
    lib = ctypes.CDLL(F.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", F.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (fmm_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_library_is_sm100a_only(F):
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(ALGS, "*.txt"))), ids=os.path.basename)
def test_library_accepts_every_algorithm_file(F, path):
    a = F.Algorithm.load(path)
    o = O.load_alg(path)
    assert (a.M, a.K, a.N, a.R) == (o.M, o.K, o.N, o.R)
    assert a.nnz == o.nnz()


def test_library_rejects_printed_strassen_W(F, tmp_path):
    # P:396-401's W fails the Brent equations (reading R1); the library must say so exactly
    f = tmp_path / "printed.txt"
    f.write_text(open(os.path.join(GOLDEN, "strassen_printed.txt")).read())
    with pytest.raises(F.FmmError) as e:
        F.Algorithm.load(str(f))
    assert e.value.status == "FMM_E_NOT_EXACT"


def test_library_create_exact_and_mutated(F):
    s = O.load_alg(os.path.join(ALGS, "laderman_class_333_23.txt"))
    a = F.Algorithm.create(3, 3, 3, 23, s.U, s.V, s.W)
    assert a.R == 23
    W = [list(r) for r in s.W]
    W[4][7] = W[4][7] + 1
    with pytest.raises(F.FmmError) as e:
        F.Algorithm.create(3, 3, 3, 23, s.U, s.V, W)
    assert e.value.status == "FMM_E_NOT_EXACT"
    # rational coefficients are accepted exactly: scale column 0 by (2, 1/4, 2)
    from fractions import Fraction as Fr
    U = [[v * (2 if r == 0 else 1) for r, v in enumerate(row)] for row in s.U]
    V = [[v * (Fr(1, 4) if r == 0 else 1) for r, v in enumerate(row)] for row in s.V]
    W = [[v * (2 if r == 0 else 1) for r, v in enumerate(row)] for row in s.W]
    F.Algorithm.create(3, 3, 3, 23, U, V, W)


def test_parser_errors_name_the_line(F, tmp_path):
    f = tmp_path / "bad.txt"
    f.write_text("# comment\n2 2 2 7 exact\n1 0 1 0 1 -1 0\n0 0 0 x 1 0 1\n")
    with pytest.raises(F.FmmError) as e:
        F.Algorithm.load(str(f))
    assert e.value.status == "FMM_E_PARSE" and "line 4" in str(e.value)
    f.write_text("2 2 2 7 apa\n")
    with pytest.raises(F.FmmError) as e:
        F.Algorithm.load(str(f))
    assert e.value.status == "FMM_E_UNSUPPORTED"


def test_hybrid_split_matches_paper(F):
    rows = [list(map(int, l.split())) for l in open(os.path.join(GOLDEN, "hybrid_split.txt")) if l.strip() and l[0] != "#"]
    for R, L, P, bfs, dfs in rows:
        assert F.hybrid_split(R, L, P) == (bfs, dfs)
    for R in (7, 15, 23, 26, 29):
        for G in (1, 2, 4, 8):
            b, d = F.hybrid_split(R, 2, G)
            assert b + d == R * R and b % G == 0 and d < G


def test_nccl_unique_id_host_only():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    a, b = F.nccl_unique_id(), F.nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b


@pytest.mark.parametrize("outer,G", [(0, 3), (1, 2), (7, 3), (12000, 8), (8192, 5)])
def test_dist_slabs_partition_the_outer_dimension(F, outer, G):
    # FMM_DIST_SLABS: rank g owns [first, last); the slabs tile [0, outer) in order, sizes differ by <= 1
    for lay, (P, N) in (("row", (outer, 5)), ("col", (5, outer))):
        spans = [F.dist_slab(P, N, lay, G, g) for g in range(G)]
        assert spans[0][0] == 0 and spans[-1][1] == outer
        assert all(spans[g][1] == spans[g + 1][0] for g in range(G - 1))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(F.FmmError):
        F.dist_slab(4, 4, "row", 2, 2)


def test_tile_map_magic_division_is_exact():
    # the leaf GEMM's tile -> task map (csrc/fmm_gemm_core.cuh, magic_div; host side make_uniform in
    # fmm_gemm_tma.cu) divides by q = umulhi(x, floor((2^32 - 1) / d)) plus ONE correction step.
    # The estimate is the quotient or one below it for every 0 <= x < 2^31: checked here on the
    # divisors' edge cases (1, powers of two, 2^k +- 1, large d) and on random pairs.
    import random
    rng = random.Random(7)

    def magic_div(x, d):
        magic = 0xFFFFFFFF // d
        q = (x * magic) >> 32
        r = x - q * d
        assert 0 <= r < 2 * d, (x, d)      # at most one correction is ever needed
        if r >= d:
            q, r = q + 1, r - d
        return q, r

    ds = [1, 2, 3, 5, 7, 8, 9, 45, 72, 80, 112, 400, 841 * 45, 2 ** 16 - 1, 2 ** 16, 2 ** 16 + 1,
          2 ** 30, 2 ** 31 - 1] + [rng.randrange(1, 2 ** 31) for _ in range(200)]
    for d in ds:
        xs = [0, 1, d - 1, d, d + 1, 2 * d - 1, 2 * d, 2 ** 31 - 1, 2 ** 31 - d] + \
             [rng.randrange(0, 2 ** 31) for _ in range(200)]
        for k in range(1, 40):                       # multiples of d and their neighbours
            xs += [k * d - 1, k * d, k * d + 1]
        for x in xs:
            if 0 <= x < 2 ** 31:
                assert magic_div(x, d) == divmod(x, d), (x, d)
