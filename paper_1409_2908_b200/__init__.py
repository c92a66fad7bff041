"""B200-native recursive fast matrix multiplication (arXiv 1409.2908): C-ABI library libfmm.so
(include/fmm.h) with sm_100a kernels, and its thin Python binding."""
import os

from .fmm import (Algorithm, Comm, DIST_SLABS, FmmError, P2P, dist_slab, Plan, dgemm, nccl_unique_id, select, hybrid_split, plan, probe_fp64_peak, shard_leaf_rows, version, LIB_PATH,  # noqa: F401
                  ROW_MAJOR, COL_MAJOR, STREAMING, WRITE_ONCE)

ALGS_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "algs")


def alg_path(name: str) -> str:
    return os.path.join(ALGS_DIR, name if name.endswith(".txt") else name + ".txt")


def load_alg(name: str) -> Algorithm:
    return Algorithm.load(alg_path(name))
