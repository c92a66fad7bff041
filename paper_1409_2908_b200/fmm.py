"""Thin ctypes binding of libfmm.so (include/fmm.h).  Argument marshalling only: every step of
the multiplication runs in the library's sm_100a kernels.  PyTorch is used for device memory and
streams; there is no CPU fallback, and a missing library raises at import time.
"""
from __future__ import annotations

import ctypes
import os
from fractions import Fraction
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
# FMM_LIB_PATH: an experiment build of the same library (build.py FMM_BUILD_VARIANT); default libfmm.so
LIB_PATH = os.environ.get("FMM_LIB_PATH") or os.path.join(_HERE, "libfmm.so")

FMM_OK = 0
_STATUS = {1: "FMM_E_INVALID_ARG", 2: "FMM_E_NOT_EXACT", 3: "FMM_E_SHAPE", 4: "FMM_E_NO_MEMORY",
           5: "FMM_E_CUDA", 6: "FMM_E_NCCL", 7: "FMM_E_UNSUPPORTED", 8: "FMM_E_PARSE"}
ROW_MAJOR, COL_MAJOR = 0, 1
STREAMING, WRITE_ONCE, PAIRWISE = 0, 1, 2
DIST_SLABS = -1  # fmm_plan_create_dist root: slab-distributed output (FMM_DIST_SLABS)
_STRATEGIES = {"streaming": STREAMING, "write_once": WRITE_ONCE, "pairwise": PAIRWISE}


class FmmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = _STATUS.get(code, str(code))


class _Options(ctypes.Structure):
    _fields_ = [("layout", ctypes.c_int), ("strategy", ctypes.c_int), ("cse", ctypes.c_int),
                ("shard_rank", ctypes.c_int), ("shard_count", ctypes.c_int),
                ("workspace_limit_bytes", ctypes.c_size_t), ("peel_align", ctypes.c_int),
                ("fuse_leaf_level", ctypes.c_int), ("shard_mode", ctypes.c_int), ("collapse_levels", ctypes.c_int),
                ("cuda_graphs", ctypes.c_int), ("peel_tiles", ctypes.c_int), ("dist_chunks", ctypes.c_int),
                ("fuse_output", ctypes.c_int), ("small_fused", ctypes.c_int), ("p2p_push", ctypes.c_int)]


# fmm_barrier_fn: int (*)(void* ctx), a host barrier over the ranks of a peer-memory plan
_BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(the CUDA library is required; there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, dp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
    p64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "fmm_alg_create": [i32, i32, i32, i32, p64, p64, p64, p64, p64, p64, ctypes.POINTER(vp)],
        "fmm_alg_load": [ctypes.c_char_p, ctypes.POINTER(vp)],
        "fmm_alg_info": [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)],
        "fmm_plan_create": [vp, i64, i64, i64, i32, ctypes.POINTER(_Options), i32, ctypes.POINTER(vp)],
        "fmm_plan": [vp, i64, i64, i64, i32, ctypes.POINTER(vp)],
        "fmm_plan_workspace_bytes": [vp, ctypes.POINTER(ctypes.c_size_t)],
        "fmm_plan_input_blocks": [vp, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_uint8), p64,
                                  ctypes.POINTER(i32)],
        "fmm_plan_stats": [vp, ctypes.POINTER(dp)],
        "fmm_plan_stats_ex": [vp, ctypes.POINTER(dp)],
        "fmm_plan_stats_ex2": [vp, ctypes.POINTER(dp), i32],
        "fmm_fused_compile_check": [vp, i32, i32, i32],
        "fmm_fused_compile_check_ex": [vp, i32, i32, i32, i32, i32],
        "fmm_alg_permute": [vp, i32, ctypes.POINTER(vp)],
        "fmm_nccl_unique_id": [ctypes.c_char_p],
        "fmm_comm_create": [ctypes.c_char_p, i32, i32, i32, ctypes.POINTER(vp)],
        "fmm_comm_info": [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)],
        "fmm_plan_create_dist": [vp, i64, i64, i64, i32, ctypes.POINTER(_Options), vp, i32, ctypes.POINTER(vp)],
        "fmm_plan_create_p2p": [vp, i64, i64, i64, i32, ctypes.POINTER(_Options), vp, i32, _BARRIER_FN, vp,
                                ctypes.POINTER(vp)],
        "fmm_plan_predict": [vp, i64, i64, i64, i32, i32, ctypes.POINTER(dp), ctypes.POINTER(i32)],
        "fmm_select": [vp, i32, i64, i64, i64, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                       ctypes.POINTER(dp)],
        "fmm_execute": [vp, vp, i64, vp, i64, vp, i64, vp],
        "fmm_exec": [vp, vp, vp, vp],
        "fmm_execute_timed": [vp, vp, i64, vp, i64, vp, i64, vp, ctypes.POINTER(ctypes.c_float)],
        "fmm_execute_host": [vp, vp, i64, vp, i64, vp, i64, vp],
        "fmm_execute_events": [vp, vp, i64, vp, i64, vp, i64, vp, ctypes.POINTER(vp)],
        "fmm_execute_profile": [vp, vp, i64, vp, i64, vp, i64, vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32),
                                ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)],
        "fmm_execute_host_async": [vp, vp, i64, vp, i64, vp, i64, vp],
        "fmm_probe_fp64_peak": [ctypes.POINTER(dp), ctypes.POINTER(dp)],
        "fmm_sync": [vp],
        "fmm_hybrid_split": [i64, i32, i64, p64, p64],
        "fmm_shard_leaf_rows": [i64, i64, i64, i64, p64, p64],
        "fmm_dist_slab": [i64, i64, i32, i32, i32, p64, p64],
        "fmm_p2p_create": [i32, i32, i32, ctypes.c_size_t, ctypes.POINTER(vp), ctypes.POINTER(vp)],
        "fmm_p2p_handle": [vp, ctypes.c_char_p],
        "fmm_p2p_open": [vp, ctypes.c_char_p],
        "fmm_p2p_reduce_slab": [vp, i64, i64, i64, vp, i64, vp],
        "fmm_dgemm": [i64, i64, i64, dp, vp, i64, vp, i64, dp, vp, i64, vp],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.fmm_alg_destroy.argtypes = [vp]
    lib.fmm_alg_destroy.restype = None
    lib.fmm_p2p_destroy.argtypes = [vp]
    lib.fmm_p2p_destroy.restype = None
    lib.fmm_plan_destroy.argtypes = [vp]
    lib.fmm_plan_destroy.restype = None
    lib.fmm_plan_options_default.argtypes = [ctypes.POINTER(_Options)]
    lib.fmm_plan_options_default.restype = None
    lib.fmm_last_error.restype = ctypes.c_char_p
    lib.fmm_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


def _check(code: int):
    if code != FMM_OK:
        raise FmmError(code, _lib.fmm_last_error().decode())


def version() -> str:
    return _lib.fmm_version().decode()


# ---- algorithms -----------------------------------------------------------------------------
class Algorithm:
    """An exact bilinear <M,K,N;R> algorithm (validated by the library's exact Brent check)."""

    def __init__(self, handle, name: str = ""):
        self._h = handle
        self.name = name
        dims = (ctypes.c_int * 4)()
        nnz = (ctypes.c_int * 3)()
        _check(_lib.fmm_alg_info(self._h, dims, nnz))
        self.M, self.K, self.N, self.R = list(dims)
        self.nnz = tuple(nnz)

    @classmethod
    def load(cls, path: str) -> "Algorithm":
        h = ctypes.c_void_p()
        _check(_lib.fmm_alg_load(path.encode(), ctypes.byref(h)))
        return cls(h, name=os.path.splitext(os.path.basename(path))[0])

    @classmethod
    def create(cls, M: int, K: int, N: int, R: int, U: Sequence, V: Sequence, W: Sequence, name: str = "") -> "Algorithm":
        """U (MK x R), V (KN x R), W (MN x R) as nested sequences of ints / Fractions."""
        def arr(X, rows):
            vals = [Fraction(v) for row in X for v in row]
            if len(vals) != rows * R:
                raise ValueError("coefficient matrix has the wrong shape")
            num = (ctypes.c_int64 * len(vals))(*[v.numerator for v in vals])
            den = (ctypes.c_int64 * len(vals))(*[v.denominator for v in vals])
            return num, den
        un, ud = arr(U, M * K)
        vn, vd = arr(V, K * N)
        wn, wd = arr(W, M * N)
        h = ctypes.c_void_p()
        _check(_lib.fmm_alg_create(M, K, N, R, un, ud, vn, vd, wn, wd, ctypes.byref(h)))
        return cls(h, name=name)

    PERMS = ["MKN", "NKM", "NMK", "KNM", "KMN", "MNK"]  # fmm_alg_permute's perm index -> base case

    def permute(self, perm: int) -> "Algorithm":
        """The equivalent algorithm for a permuted base case (Props. 1-2, fmm_alg_permute)."""
        h = ctypes.c_void_p()
        _check(_lib.fmm_alg_permute(self._h, perm, ctypes.byref(h)))
        return Algorithm(h, name=f"{self.name}^{self.PERMS[perm]}")

    def predict_ms(self, P: int, Q: int, N: int, levels: int, layout: str = "row") -> float:
        """The library's cost model (fmm_plan_predict): predicted ms of the plan on one B200."""
        ms, used = ctypes.c_double(), ctypes.c_int()
        _check(_lib.fmm_plan_predict(self._h, P, Q, N, levels, ROW_MAJOR if layout == "row" else COL_MAJOR,
                                     ctypes.byref(ms), ctypes.byref(used)))
        return ms.value

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fmm_alg_destroy(self._h)
            self._h = None


def select(algs: Sequence[Algorithm], P: int, Q: int, N: int, max_levels: int = 3, layout: str = "row"):
    """Shape matching (fmm_select): (algorithm or None for classical, levels, predicted ms) with the
    algorithm already permuted to the chosen base case."""
    arr = (ctypes.c_void_p * max(1, len(algs)))(*[a._h for a in algs])
    ai, pm, lv, ms = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    _check(_lib.fmm_select(arr, len(algs), P, Q, N, max_levels, ROW_MAJOR if layout == "row" else COL_MAJOR,
                           ctypes.byref(ai), ctypes.byref(pm), ctypes.byref(lv), ctypes.byref(ms)))
    if ai.value < 0:
        return None, 0, ms.value
    return algs[ai.value].permute(pm.value), lv.value, ms.value


# ---- tensors --------------------------------------------------------------------------------
def _mat(t, layout: int, rows: int, cols: int, what: str):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2:
        raise TypeError(f"{what} must be a 2-D float64 CUDA tensor")
    if tuple(t.shape) != (rows, cols):
        raise ValueError(f"{what} has shape {tuple(t.shape)}, expected {(rows, cols)}")
    s0, s1 = t.stride()
    if layout == ROW_MAJOR:
        if s1 != 1 and cols > 1:
            raise ValueError(f"{what} must be row-major (unit column stride)")
        ld = s0 if rows > 1 else max(cols, 1)
    else:
        if s0 != 1 and rows > 1:
            raise ValueError(f"{what} must be column-major (unit row stride)")
        ld = s1 if cols > 1 else max(rows, 1)
    return ctypes.c_void_p(t.data_ptr()), int(max(ld, 1))


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ---- multi-GPU -------------------------------------------------------------------------------
def nccl_unique_id() -> bytes:
    """fmm_nccl_unique_id: 128 bytes for rank 0 to share with every rank."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.fmm_nccl_unique_id(buf))
    return buf.raw


class Comm:
    """An NCCL communicator owned by the library (fmm_comm_create), one rank per process and GPU."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: Optional[int] = None):
        import torch
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _check(_lib.fmm_comm_create(ctypes.create_string_buffer(uid, 128), nranks, rank, self.device, ctypes.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    @classmethod
    def from_torch_distributed(cls, group=None, device: Optional[int] = None) -> "Comm":
        """Bootstrap through an initialised torch.distributed group (rank 0's id is broadcast)."""
        import torch.distributed as dist
        obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], dist.get_world_size(group), dist.get_rank(group), device)

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fmm_comm_destroy(self._h)
            self._h = None


# ---- plans ----------------------------------------------------------------------------------
class Plan:
    """C (P x N) = A (P x Q) @ B (Q x N) with `levels` recursive steps of `alg` (fmm_plan_create)."""

    def __init__(self, alg: Algorithm, P: int, Q: int, N: int, levels: int, layout: str = "row",
                 strategy: str = "streaming", cse: bool = True, shard_rank: int = 0, shard_count: int = 1,
                 device: Optional[int] = None, workspace_limit_bytes: int = 0, peel_align: bool = True,
                 fuse=False, collapse: bool = True, comm: Optional[Comm] = None, root: int = 0,
                 shard_mode: str = "leaf", cuda_graphs: bool = True, peel_tiles: bool = False,
                 p2p: Optional["P2P"] = None, barrier=None, dist_chunks: Optional[int] = None,
                 fuse_output: Optional[bool] = None, small: Optional[bool] = None,
                 p2p_push: Optional[bool] = None):
        """comm: an NCCL Comm -> fmm_plan_create_dist (the reduce runs inside execute, in dist_chunks
        overlapped row chunks where it applies).  p2p + barrier: a P2P object and a zero-argument host
        barrier over the same ranks (e.g. torch.distributed.barrier) -> fmm_plan_create_p2p (the
        peer-memory combine runs inside execute, which then blocks).  root: the rank that receives C,
        or "slabs" for slab-distributed output.  fuse: False / 0 separate leaf-level launches, True / 1
        the fused leaf level with addition CTAs, 2 or "bg" the fused leaf level with the jobs in the
        GEMM CTAs' spare warps (fuse_leaf_level, fmm.h)."""
        import torch
        self.alg, self.P, self.Q, self.N, self.levels = alg, P, Q, N, levels
        self.layout = ROW_MAJOR if layout == "row" else COL_MAJOR
        o = _Options()
        _lib.fmm_plan_options_default(ctypes.byref(o))
        o.layout = self.layout
        if strategy not in _STRATEGIES:
            raise ValueError(f"strategy must be one of {sorted(_STRATEGIES)}")
        o.strategy = _STRATEGIES[strategy]
        o.cuda_graphs = int(bool(cuda_graphs))
        o.peel_tiles = int(bool(peel_tiles))
        o.cse = int(bool(cse))
        o.shard_rank, o.shard_count = shard_rank, shard_count
        o.workspace_limit_bytes = workspace_limit_bytes
        o.peel_align = int(bool(peel_align))
        o.fuse_leaf_level = 2 if fuse in (2, "bg") else int(bool(fuse))
        o.collapse_levels = int(bool(collapse))
        o.shard_mode = {"leaf": 0, "top": 1}[shard_mode]
        if dist_chunks is not None:
            o.dist_chunks = int(dist_chunks)
        if fuse_output is not None:
            o.fuse_output = int(bool(fuse_output))
        if small is not None:
            o.small_fused = int(bool(small))
        if p2p_push is not None:
            o.p2p_push = int(bool(p2p_push))
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        self.comm = comm  # a distributed plan keeps its communicator / peer buffers alive
        self.p2p = p2p
        if root == "slabs":
            root = DIST_SLABS
        if comm is not None and p2p is not None:
            raise ValueError("a plan combines through NCCL (comm) or peer memory (p2p), not both")
        if p2p is not None:
            if barrier is None:
                raise ValueError("a peer-memory plan needs a host barrier over its ranks")

            def _bar(_ctx):
                try:
                    barrier()
                    return 0
                except Exception:  # noqa: BLE001  (reported to the library as a failed barrier)
                    return 1
            self._barrier = _BARRIER_FN(_bar)  # kept alive as long as the plan
            self.device = p2p.device
            _check(_lib.fmm_plan_create_p2p(alg._h, P, Q, N, levels, ctypes.byref(o), p2p._h, root, self._barrier,
                                            None, ctypes.byref(h)))
        elif comm is None:
            _check(_lib.fmm_plan_create(alg._h, P, Q, N, levels, ctypes.byref(o), self.device, ctypes.byref(h)))
        else:
            self.device = comm.device
            _check(_lib.fmm_plan_create_dist(alg._h, P, Q, N, levels, ctypes.byref(o), comm._h, root, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fmm_plan_destroy(self._h)
            self._h = None

    @property
    def workspace_bytes(self) -> int:
        b = ctypes.c_size_t()
        _check(_lib.fmm_plan_workspace_bytes(self._h, ctypes.byref(b)))
        return b.value

    def input_blocks(self):
        """(needA, needB, (P', Q', N'), need_all): the top-level blocks of A (M*K flags, row-major over
        the block grid) and B (K*N) this plan reads (fmm_plan_input_blocks)."""
        a = self.alg
        na = (ctypes.c_uint8 * (a.M * a.K))()
        nb = (ctypes.c_uint8 * (a.K * a.N))()
        core = (ctypes.c_int64 * 3)()
        allf = ctypes.c_int()
        _check(_lib.fmm_plan_input_blocks(self._h, na, nb, core, ctypes.byref(allf)))
        return [bool(x) for x in na], [bool(x) for x in nb], tuple(core), bool(allf.value)

    def stats(self) -> dict:
        s = (ctypes.c_double * 19)()
        _check(_lib.fmm_plan_stats_ex2(self._h, s, 19))
        keys = ["gemm_flops", "add_flops", "add_bytes", "gemm_bytes", "launches", "levels", "leaves", "paper_flops",
                "leaf_flops", "fused_add_bytes", "fused_launches", "formation_bytes", "assembly_bytes", "strip_flops",
                "collapsed", "tiled_peel", "fused_output", "collapsed_assembly", "small_fused"]
        return dict(zip(keys, list(s)))

    def new_output(self):
        import torch
        if self.layout == ROW_MAJOR:
            return torch.empty(self.P, self.N, dtype=torch.float64, device=f"cuda:{self.device}")
        return torch.empty(self.N, self.P, dtype=torch.float64, device=f"cuda:{self.device}").t()

    def _args(self, A, B, C):
        a, lda = _mat(A, self.layout, self.P, self.Q, "A")
        b, ldb = _mat(B, self.layout, self.Q, self.N, "B")
        c, ldc = _mat(C, self.layout, self.P, self.N, "C")
        return a, lda, b, ldb, c, ldc

    def execute(self, A, B, C=None, stream=None):
        """C <- A @ B on the stream (asynchronous). Returns C."""
        if C is None:
            C = self.new_output()
        _check(_lib.fmm_execute(self._h, *self._args(A, B, C), _stream_ptr(stream)))
        return C

    def execute_timed(self, A, B, C=None, stream=None):
        """Blocking, plain launches with an event after each (fmm_execute_timed); returns
        (C, {formation, gemm (leaf products), assembly, strips (peel GEMMs), total} ms), total
        including a distributed plan's combine."""
        if C is None:
            C = self.new_output()
        ms = (ctypes.c_float * 5)()
        _check(_lib.fmm_execute_timed(self._h, *self._args(A, B, C), _stream_ptr(stream), ms))
        return C, {"formation_ms": ms[0], "gemm_ms": ms[1], "assembly_ms": ms[2], "strips_ms": ms[3],
                   "total_ms": ms[4]}

    KINDS = ["form_A", "form_B", "leaf_gemm", "assembly", "strips", "thin", "fused_leaf_level", "combine", "zero",
             "small_fused"]

    def execute_profile(self, A, B, C=None, stream=None, max_launches=256):
        """Blocking diagnostic execute (fmm_execute_profile): [(kind, level, ms)] per launch."""
        if C is None:
            C = self.new_output()
        kind = (ctypes.c_int * max_launches)()
        level = (ctypes.c_int * max_launches)()
        ms = (ctypes.c_float * max_launches)()
        n = ctypes.c_int()
        _check(_lib.fmm_execute_profile(self._h, *self._args(A, B, C), _stream_ptr(stream), max_launches, kind, level,
                                        ms, ctypes.byref(n)))
        return [(self.KINDS[kind[q]] if 0 <= kind[q] < len(self.KINDS) else str(kind[q]), level[q], ms[q])
                for q in range(min(n.value, max_launches))]

    def execute_events(self, A, B, C, events, stream=None):
        """Asynchronous execute that records 4 torch.cuda.Event on the stream: before, after
        formation, after the leaf GEMM, after assembly/strips."""
        ev = (ctypes.c_void_p * 4)(*[e.cuda_event for e in events])
        _check(_lib.fmm_execute_events(self._h, *self._args(A, B, C), _stream_ptr(stream), ev))
        return C

    def execute_host(self, A, B, C, stream=None, asynchronous=False):
        """Host (CPU) tensors / arrays in, host result out: H2D, execute, D2H.  Blocking unless
        asynchronous=True (fmm_execute_host_async: pipelined with neighbouring calls; the host
        buffers must be pinned and stay untouched until sync())."""
        import numpy as np
        import torch

        def hp(x, rows, cols, what, writable=False):
            # the same layout rules as _mat(): unit stride along the contiguous dimension, a
            # non-negative leading dimension, and a writeable output (the library copies whole
            # rows / columns of ld-strided storage, so any other view would be read or written wrongly)
            if isinstance(x, torch.Tensor):
                if x.is_cuda or x.dtype != torch.float64 or x.dim() != 2:
                    raise TypeError(f"{what} must be a 2-D float64 CPU tensor")
                s0, s1 = x.stride()
                ptr = x.data_ptr()
            else:
                if not isinstance(x, np.ndarray) or x.dtype != np.float64 or x.ndim != 2:
                    raise TypeError(f"{what} must be a 2-D float64 array")
                if x.strides[0] % 8 or x.strides[1] % 8:
                    raise ValueError(f"{what} has strides that are not whole elements")
                s0, s1 = x.strides[0] // 8, x.strides[1] // 8
                ptr = x.ctypes.data
                if writable and not x.flags.writeable:
                    raise ValueError(f"{what} is read-only")
            if tuple(x.shape) != (rows, cols):
                raise ValueError(f"{what} has shape {tuple(x.shape)}, expected {(rows, cols)}")
            if s0 < 0 or s1 < 0:
                raise ValueError(f"{what} has a negative stride")
            if self.layout == ROW_MAJOR:
                if s1 != 1 and cols > 1:
                    raise ValueError(f"{what} must be row-major (unit column stride)")
                ld = s0 if rows > 1 else max(cols, 1)
            else:
                if s0 != 1 and rows > 1:
                    raise ValueError(f"{what} must be column-major (unit row stride)")
                ld = s1 if cols > 1 else max(rows, 1)
            return ctypes.c_void_p(ptr), int(max(ld, 1))
        a, lda = hp(A, self.P, self.Q, "A")
        b, ldb = hp(B, self.Q, self.N, "B")
        c, ldc = hp(C, self.P, self.N, "C", True)
        fn = _lib.fmm_execute_host_async if asynchronous else _lib.fmm_execute_host
        _check(fn(self._h, a, lda, b, ldb, c, ldc, _stream_ptr(stream)))
        return C

    def sync(self):
        _check(_lib.fmm_sync(self._h))


def plan(alg: Algorithm, M: int, K: int, N: int, levels: int) -> Plan:
    """The north-star spelling fmm_plan(alg, M, K, N, levels): default options, row-major."""
    return Plan(alg, M, K, N, levels)


def dgemm(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, stream=None):
    """C = alpha A B + beta C with the library's DMMA GEMM kernel (row-major CUDA tensors)."""
    import torch
    m, k = A.shape
    n = B.shape[1]
    if C is None:
        C = torch.empty(m, n, dtype=torch.float64, device=A.device)
    a, lda = _mat(A, ROW_MAJOR, m, k, "A")
    b, ldb = _mat(B, ROW_MAJOR, k, n, "B")
    c, ldc = _mat(C, ROW_MAJOR, m, n, "C")
    _check(_lib.fmm_dgemm(m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, _stream_ptr(stream)))
    return C


def fused_compile_check(alg: "Algorithm", layout: str = "row", cse: bool = True, bn: int = 128, ks: int = 16,
                        mode: int = 1) -> None:
    """NVRTC-compile the fused leaf-level kernel of `alg` (host only; raises FmmError on failure) for
    ring depth `ks` and fuse_leaf_level `mode` (1 addition CTAs, 2 background jobs)."""
    _check(_lib.fmm_fused_compile_check_ex(alg._h, ROW_MAJOR if layout == "row" else COL_MAJOR, int(bool(cse)), bn, ks,
                                           mode))


def probe_fp64_peak():
    """(DMMA TFLOP/s, DFMA TFLOP/s) measured on the current device by the library's probes."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(_lib.fmm_probe_fp64_peak(ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def shard_leaf_rows(leaves: int, rows: int, G: int, g: int):
    """[(r0, r1)] per leaf: the rows of each leaf product that worker g of G computes."""
    r0 = (ctypes.c_int64 * leaves)()
    r1 = (ctypes.c_int64 * leaves)()
    _check(_lib.fmm_shard_leaf_rows(leaves, rows, G, g, r0, r1))
    return list(zip(r0, r1))


class _CudaBuffer:
    """A raw device allocation seen by torch through __cuda_array_interface__ (no copy)."""

    def __init__(self, ptr: int, shape, owner):
        self.owner = owner  # keeps the allocation alive while a tensor views it
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8", "data": (ptr, False),
                                         "version": 3, "strides": None}


class P2P:
    """The multi-GPU combine over peer memory (fmm_p2p_*): each rank's partial C
    lives in a library buffer mapped into every peer by CUDA IPC, and reduce_slab sums this rank's
    slab of all partials in ONE kernel (pull-based reduce-scatter, no NCCL in the data path).  The
    caller orders the ranks: all partials written (synchronise + barrier) before any reduce_slab,
    all reduces finished before a partial is overwritten."""

    def __init__(self, nranks: int, rank: int, nbytes: int, device: Optional[int] = None):
        import torch
        self.nranks, self.rank = nranks, rank
        self.device = torch.cuda.current_device() if device is None else device
        h, local = ctypes.c_void_p(), ctypes.c_void_p()
        _check(_lib.fmm_p2p_create(nranks, rank, self.device, nbytes, ctypes.byref(h), ctypes.byref(local)))
        self._h, self.local_ptr, self.nbytes = h, local.value, nbytes

    def handle(self) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _check(_lib.fmm_p2p_handle(self._h, buf))
        return buf.raw

    def open(self, handles) -> None:
        """Map every rank's partial (handles: one 64-byte handle per rank, rank order)."""
        if len(handles) != self.nranks or any(len(x) != 64 for x in handles):
            raise ValueError("need one 64-byte handle per rank")
        blob = b"".join(handles)
        _check(_lib.fmm_p2p_open(self._h, ctypes.create_string_buffer(blob, len(blob))))

    @classmethod
    def from_torch_distributed(cls, nbytes: int, group=None, device: Optional[int] = None) -> "P2P":
        import torch.distributed as dist
        p = cls(dist.get_world_size(group), dist.get_rank(group), nbytes, device)
        hs = [None] * p.nranks
        dist.all_gather_object(hs, p.handle(), group=group)
        p.open(hs)
        return p

    def partial(self, P: int, N: int, layout: str = "row"):
        """The P x N partial-product view (row- or column-major) over this rank's buffer: the C
        to pass to the shard plan's execute."""
        import torch
        if 8 * P * N > self.nbytes:
            raise ValueError("the buffer is smaller than P x N doubles")
        if layout == "row":
            return torch.as_tensor(_CudaBuffer(self.local_ptr, (P, N), self), device=f"cuda:{self.device}")
        return torch.as_tensor(_CudaBuffer(self.local_ptr, (N, P), self), device=f"cuda:{self.device}").t()

    def reduce_slab(self, outer: int, inner: int, out, ld: Optional[int] = None, stream=None):
        """out (this rank's fmm_dist_slab rows of the outer x inner partial storage, a float64 CUDA
        tensor with unit column stride) <- the sum over ranks.  Asynchronous on the stream."""
        if out.dtype != torch_float64() or not out.is_cuda or (out.dim() == 2 and out.shape[0] > 1 and out.stride(1) != 1):
            raise TypeError("out must be a float64 CUDA tensor with unit column stride")
        ldo = out.stride(0) if out.dim() == 2 else inner
        _check(_lib.fmm_p2p_reduce_slab(self._h, outer, inner, inner if ld is None else ld,
                                        ctypes.c_void_p(out.data_ptr()), ldo, _stream_ptr(stream)))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.fmm_p2p_destroy(self._h)
            self._h = None


def torch_float64():
    import torch
    return torch.float64


def dist_slab(P: int, N: int, layout: str, nranks: int, rank: int):
    """(first, last): the rows (row-major) or columns (column-major) of C that `rank` holds after a
    slab-distributed combine (root="slabs"; fmm_dist_slab)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.fmm_dist_slab(P, N, ROW_MAJOR if layout == "row" else COL_MAJOR, nranks, rank, ctypes.byref(a),
                              ctypes.byref(b)))
    return a.value, b.value


def hybrid_split(R: int, L: int, G: int):
    bfs, dfs = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.fmm_hybrid_split(R, L, G, ctypes.byref(bfs), ctypes.byref(dfs)))
    return bfs.value, dfs.value
