"""Multi-GPU plumbing for the leaf-sharded plan (one process per GPU, torch.distributed).

Each rank runs a plan with shard_rank = rank, shard_count = world (HYBRID arithmetic, P:823-829,
with GPUs in place of threads) and holds a partial C; the C_k combination is linear in the
partials, so C = sum over ranks, done as one NCCL reduce (sum, fp64) to the root.
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
