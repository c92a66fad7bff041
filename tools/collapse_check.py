import os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import fmm_inputs as I
import paper_1409_2908_b200 as F
from oracle import oracle as O
for name, P, Q, N, L, lay in [("strassen_222_7", 256, 256, 256, 2, "row"), ("winograd_class_222_7", 1024, 1024, 1024, 2, "col"),
                              ("strassen_222_7", 1000, 998, 1002, 3, "row"), ("winograd_class_222_7", 2048, 512, 1536, 2, "row")]:
    A, B = I.problem(P, Q, N, seed=1)
    def dev(x):
        return torch.from_numpy(np.ascontiguousarray(x)).cuda() if lay == "row" else torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    res = {}
    for col in (True, False):
        p = F.Plan(F.load_alg(name), P, Q, N, L, layout=lay, cse=False, collapse=col)
        C = p.execute(dev(A), dev(B)); torch.cuda.synchronize()
        res[col] = (C.cpu().numpy(), p.stats())
    ref = O.fast(A, B, O.load_alg(F.alg_path(name)), L)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    Ai, Bi = I.problem(P, Q, N, seed=2, kind="integers")
    p = F.Plan(F.load_alg(name), P, Q, N, L, layout=lay)
    Ci = p.execute(dev(Ai), dev(Bi)).cpu().numpy()
    print(name, P, Q, N, L, lay, "collapsed==separate", np.array_equal(res[True][0], res[False][0]),
          "err", np.max(np.abs(res[True][0] - ref)) / nrm, "bytes", res[True][1]["add_bytes"] / 1e9, "vs", res[False][1]["add_bytes"] / 1e9,
          "launches", res[True][1]["launches"], res[False][1]["launches"], "int exact", np.array_equal(Ci, Ai @ Bi), flush=True)
