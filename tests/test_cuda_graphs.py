"""CUDA-graph replay of a plan's launch sequence (plan option cuda_graphs, the default): the second
execute with a cached A/B/C pointer set captures the launches into a graph, later ones replay it.
Replays must read the buffers' current contents (new data in the same buffers gives the new
product), survive slot eviction (a third pointer set rebuilds a slot and drops its graph) and run
on any stream, bitwise equal to plain launches."""
import numpy as np
import pytest

import fmm_inputs as I

pytestmark = pytest.mark.gpu


def _F():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    return F


@pytest.mark.parametrize("name,P,Q,N,L,layout,strategy", [
    ("winograd_class_222_7", 512, 512, 512, 2, "col", "streaming"),   # collapsed levels
    ("alg_424_26", 328, 66, 330, 2, "row", "streaming"),               # peeling, strips
    ("hk_class_323_15", 100, 60, 90, 1, "row", "pairwise"),            # several launches per chain
    ("strassen_222_7", 40, 36, 44, 3, "row", "write_once"),            # thin skinny strips
])
def test_graph_replay_matches_plain_launches(name, P, Q, N, L, layout, strategy):
    import torch
    F = _F()

    def dev(x):
        if layout == "row":
            return torch.from_numpy(np.ascontiguousarray(x)).cuda()
        return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()

    g = F.Plan(F.load_alg(name), P, Q, N, L, layout=layout, strategy=strategy)
    plain = F.Plan(F.load_alg(name), P, Q, N, L, layout=layout, strategy=strategy, cuda_graphs=False)
    A, B = dev(np.zeros((P, Q))), dev(np.zeros((Q, N)))
    C = g.new_output()
    s = torch.cuda.Stream()
    for it in range(5):  # run 0 plain, run 1 captures, runs 2-4 replay
        An, Bn = I.problem(P, Q, N, seed=100 + it, kind="integers")
        A.copy_(torch.from_numpy(An)); B.copy_(torch.from_numpy(Bn))
        stream = s if it % 2 else None
        g.execute(A, B, C, stream=stream)
        ref = plain.execute(A, B)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), An @ Bn), it
        assert np.array_equal(C.cpu().numpy(), ref.cpu().numpy()), it


def test_graph_slots_evicted_and_rebuilt():
    import torch
    F = _F()
    P = Q = N = 256
    p = F.Plan(F.load_alg("strassen_222_7"), P, Q, N, 2)
    sets = []
    for k in range(3):
        An, Bn = I.problem(P, Q, N, seed=200 + k, kind="integers")
        sets.append((torch.from_numpy(An).cuda(), torch.from_numpy(Bn).cuda(), p.new_output(), An @ Bn))
    order = [0, 0, 0, 1, 1, 1, 2, 2, 0, 0, 1, 2, 2, 2, 0]
    for k in order:
        A, B, C, want = sets[k]
        C.zero_()
        p.execute(A, B, C)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), want), k


def test_host_async_with_graphs():
    # fmm_execute_host_async alternates two staging sets: each gets its own slot and graph
    import torch
    F = _F()
    P, Q, N = 300, 200, 250
    p = F.Plan(F.load_alg("winograd_class_222_7"), P, Q, N, 2)
    for it in range(5):
        An, Bn = I.problem(P, Q, N, seed=300 + it, kind="integers")
        C = np.zeros((P, N))
        p.execute_host(An, Bn, C)
        assert np.array_equal(C, An @ Bn), it
