"""Multi-process (world_size 2 and 3, gloo, CPU) check of the N > 1 path's host side:
the library's leaf partition (HYBRID arithmetic) covers every row of every leaf
exactly once across ranks, and the partial products combined by the same combine_partials used
by bench.py (one reduce) give exactly A*B.  The per-rank partial product here is a small exact
integer evaluation of one recursion level written in the test (the GPU path is covered by
tests/test_gpu_parity.py::test_shards_sum_to_product)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ALGS, ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, alg_name, q, mode="root"):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import fmm_inputs as I
        import paper_1409_2908_b200 as F
        from paper_1409_2908_b200.dist import combine_partials, scatter_partials
        from oracle import oracle as O
        a = O.load_alg(os.path.join(ALGS, alg_name + ".txt"))
        U, V, W = (np.array(X, dtype=np.float64) for X in a.as_float())
        M, K, N, R = a.M, a.K, a.N, a.R
        p, qd, n = 5, 3, 4
        A, B = I.problem(M * p, K * qd, N * n, seed=3, kind="integers")
        own = F.shard_leaf_rows(R, p, world, rank)
        C = np.zeros((M * p, N * n))
        for r in range(R):
            r0, r1 = own[r]
            if r1 <= r0:
                continue
            S = sum(U[i, r] * A[(i // K) * p:(i // K + 1) * p, (i % K) * qd:(i % K + 1) * qd] for i in range(M * K))
            T = sum(V[j, r] * B[(j // N) * qd:(j // N + 1) * qd, (j % N) * n:(j % N + 1) * n] for j in range(K * N))
            Mr = np.zeros((p, n))
            Mr[r0:r1] = S[r0:r1] @ T
            for k in range(M * N):
                C[(k // N) * p:(k // N + 1) * p, (k % N) * n:(k % N + 1) * n] += W[k, r] * Mr
        owns = [None] * world
        dist.all_gather_object(owns, own)
        if mode != "root":
            # slab-distributed output: row slabs of a row-major C, column slabs of a column-major C
            Ct = torch.from_numpy(C) if mode == "slabs_row" else torch.from_numpy(np.ascontiguousarray(C.T)).t()
            first, last = scatter_partials(Ct)
            lay = "row" if mode == "slabs_row" else "col"
            assert (first, last) == F.dist_slab(C.shape[0], C.shape[1], lay, world, rank)
            want = A @ B
            got = Ct.numpy()
            ok = np.array_equal(got[first:last], want[first:last]) if lay == "row" else \
                np.array_equal(got[:, first:last], want[:, first:last])
            ok_all = [None] * world
            dist.all_gather_object(ok_all, ok)
            if rank == 0:
                q.put((all(ok_all), True))
            return
        Ct = torch.from_numpy(C)
        combine_partials(Ct, root=0)
        if rank == 0:
            cover = np.zeros((R, p), dtype=int)
            for o in owns:
                for z, (r0, r1) in enumerate(o):
                    cover[z, r0:r1] += 1
            q.put((bool(np.array_equal(Ct.numpy(), A @ B)), bool((cover == 1).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,alg,mode", [(2, "strassen_222_7", "root"), (3, "hk_class_323_15", "root"),
                                           (2, "alg_433_29", "root"), (3, "alg_424_26", "slabs_row"),
                                           (2, "hk_class_323_15", "slabs_col")])
def test_sharded_partials_reduce_to_product(world, alg, mode):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, alg, q, mode)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs)
    exact, covered = q.get(timeout=5)
    assert covered, "leaf rows not partitioned exactly once"
    assert exact, "reduced partials differ from A*B"
