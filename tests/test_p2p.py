"""The combine over peer memory (fmm_p2p_*): world-size 2 and 3 processes, each
with its HYBRID leaf shard written into its IPC-exported partial buffer, then ONE
reduce kernel per rank pulling its slab from every rank's partial -- called by hand
(fmm_p2p_reduce_slab) and inside fmm_execute of the library's peer-memory plan
(fmm_plan_create_p2p, root and slab output; and the push mode, p2p_push, where the kernels that
write C store each rank's partial straight into the root's buffer).  The ranks share the one GPU of
this box (CUDA IPC works between processes on one device), gloo carries only the handle exchange
and the two barriers; no kernel waits on another rank's kernel.  Integer inputs: the slabs must
equal the exact product bit for bit, in both layouts."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, layout, alg_name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = False
    try:
        import fmm_inputs as I
        import paper_1409_2908_b200 as F
        torch.cuda.set_device(0)
        P, Q, N = 300, 200, 250
        A, B = I.problem(P, Q, N, seed=31, kind="integers")

        def dev(x):
            if layout == "row":
                return torch.from_numpy(np.ascontiguousarray(x)).cuda()
            return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
        p2p = F.P2P.from_torch_distributed(8 * P * N)
        plan = F.Plan(F.load_alg(alg_name), P, Q, N, 2, layout=layout, shard_rank=rank, shard_count=world)
        C = p2p.partial(P, N, layout)
        for it in range(2):  # twice: the buffers are reused across executes
            plan.execute(dev(A), dev(B), C)
            torch.cuda.synchronize()
            dist.barrier()  # every partial complete
            outer, inner = (P, N) if layout == "row" else (N, P)
            r0, r1 = F.dist_slab(P, N, layout, world, rank)
            out = torch.empty(r1 - r0, inner, dtype=torch.float64, device="cuda")
            p2p.reduce_slab(outer, inner, out)
            torch.cuda.synchronize()
            dist.barrier()  # every reduce done before a partial is overwritten
            want = (A @ B)[r0:r1] if layout == "row" else (A @ B)[:, r0:r1].T
            ok = bool(np.array_equal(out.cpu().numpy(), want))
            if not ok:
                break
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if rank == 0:
            q.put(all(oks))
        del C, plan
        dist.barrier()
        del p2p
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout,alg", [(2, "row", "winograd_class_222_7"), (3, "col", "alg_424_26"),
                                              (2, "col", "hk_class_323_15")])
def test_p2p_slab_combine(world, layout, alg):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, layout, alg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    assert q.get(timeout=5), "reduced slabs differ from A*B"


def _plan_worker(rank, world, port, layout, alg_name, root, q, push=False):
    # the library's own combine: fmm_plan_create_p2p, the reduce inside fmm_execute, the host
    # barrier supplied as a callback (gloo's torch.distributed.barrier)
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import fmm_inputs as I
        import paper_1409_2908_b200 as F
        torch.cuda.set_device(0)
        P, Q, N = 301, 200, 250  # odd P: a peel strip at the top level
        A, B = I.problem(P, Q, N, seed=37, kind="integers")

        def dev(x):
            if layout == "row":
                return torch.from_numpy(np.ascontiguousarray(x)).cuda()
            return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
        # push mode: every rank's buffer holds G partial slots (16-byte aligned), the root's receives them
        p2p = F.P2P.from_torch_distributed(8 * ((P * N + 1) // 2 * 2) * (world if push else 1))
        plan = F.Plan(F.load_alg(alg_name), P, Q, N, 2, layout=layout, p2p=p2p, barrier=dist.barrier, root=root,
                      p2p_push=push)
        want = A @ B
        ok = True
        for it in range(3):  # the partial buffers are reused across executes
            C = torch.full((P, N), float("nan"), dtype=torch.float64, device="cuda") if layout == "row" else \
                torch.full((N, P), float("nan"), dtype=torch.float64, device="cuda").t()
            plan.execute(dev(A), dev(B), C)
            torch.cuda.synchronize()
            got = C.cpu().numpy()
            if root == "slabs":
                r0, r1 = F.dist_slab(P, N, layout, world, rank)
                ok &= bool(np.array_equal(got[r0:r1], want[r0:r1]) if layout == "row" else
                           np.array_equal(got[:, r0:r1], want[:, r0:r1]))
            elif rank == root:
                ok &= bool(np.array_equal(got, want))
            else:  # other ranks' C is left untouched
                ok &= bool(np.isnan(got).all())
        oks = [None] * world
        dist.all_gather_object(oks, ok)
        if rank == 0:
            q.put(all(oks))
        del plan
        dist.barrier()
        del p2p
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,layout,alg,root,push", [(2, "row", "winograd_class_222_7", 0, False),
                                                        (2, "col", "hk_class_323_15", 1, False),
                                                        (3, "row", "alg_424_26", "slabs", False),
                                                        (2, "col", "strassen_222_7", "slabs", False),
                                                        # push mode (p2p_push): the partials are stored into
                                                        # the root's slots by the kernels that write C
                                                        (2, "row", "winograd_class_222_7", 0, True),
                                                        (3, "col", "alg_424_26", 2, True),
                                                        (3, "row", "hk_class_323_15", 1, True),
                                                        # slab output with p2p_push: the pull path
                                                        (2, "row", "strassen_222_7", "slabs", True)])
def test_p2p_plan_combines_inside_execute(world, layout, alg, root, push):
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, layout, alg, root, q, push)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    assert q.get(timeout=5), "the combined C differs from A*B"


@pytest.mark.parametrize("workload,extra", [("c1", []), ("c3", ["--shard-mode", "top", "--output", "slabs"]),
                                            ("c1", ["--shard-mode", "slab"]), ("c3", ["--combine", "p2p_push"])])
def test_bench_two_ranks_on_one_gpu(workload, extra):
    # `bench.py --gpus 2` with no torchrun wrapper launches the two ranks itself; with gloo they share
    # this GPU and the peer-memory plan combines inside fmm_execute (a control-flow check: the line
    # says it is not a measurement)
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo",
                        "--workload", workload, "--steps", "3", "--warmup", "3", "--no-cpu", "--no-other", *extra],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    want = "no combine" if "slab" in extra else "peer-memory combine inside fmm_execute"
    assert line["n_gpus"] == 2 and want in line["config"]["parallelism"]
    assert "NOT a measurement" in line["config"]["dist_backend"]
    assert line["result_check"]["ok"]
