"""Multi-GPU plumbing for the leaf-sharded plan (one process per GPU, torch.distributed).

Each rank runs a plan with shard_rank = rank, shard_count = world (HYBRID arithmetic, P:823-829,
with GPUs in place of threads) and holds a partial C; the C_k combination is linear in the
partials, so C = sum over ranks, done as one NCCL reduce (sum, fp64) to the root, or (scatter_partials) as one reduce per slab of C onto its owning rank.
"""
import torch
import torch.distributed as dist


def storage_view(C: torch.Tensor) -> torch.Tensor:
    """The contiguous tensor behind a row- or column-major C (collectives need contiguity)."""
    if C.is_contiguous():
        return C
    if C.t().is_contiguous():
        return C.t()
    raise ValueError("C must be row- or column-major without gaps")


def combine_partials(C: torch.Tensor, root: int = 0, group=None) -> torch.Tensor:
    """Sum the ranks' partial products into C on `root` (in place)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.reduce(storage_view(C), dst=root, op=dist.ReduceOp.SUM, group=group)
    return C


def slab_range(outer: int, world: int, rank: int):
    """Rows [first, last) of the contiguous storage that `rank` owns (fmm_dist_slab's split)."""
    return outer * rank // world, outer * (rank + 1) // world


def scatter_partials(C: torch.Tensor, group=None):
    """Slab-distributed combine (reduce-scatter): slab g of C's contiguous storage
    (rows of a row-major C, columns of a column-major one) is summed onto rank g, as the library's
    FMM_DIST_SLABS does with grouped ncclReduce calls.  Returns this rank's (first, last)."""
    S = storage_view(C)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return 0, S.shape[0]
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    for g in range(world):
        r0, r1 = slab_range(S.shape[0], world, g)
        if r1 > r0:
            dist.reduce(S[r0:r1], dst=dist.get_global_rank(group, g) if group is not None else g,
                        op=dist.ReduceOp.SUM, group=group)
    return slab_range(S.shape[0], world, rank)
