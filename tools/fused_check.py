"""Quick GPU check of the fused leaf level: fused vs unfused (cse off: same chain order, bitwise
equal) and vs the oracle, on several algorithms / shapes / layouts."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fmm_inputs as I  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = [("strassen_222_7", 256, 256, 256, 1, "row"), ("strassen_222_7", 512, 384, 640, 2, "row"),
         ("winograd_class_222_7", 1024, 1024, 1024, 2, "col"), ("hk_class_323_15", 1203, 602, 1205, 2, "row"),
         ("alg_424_26", 1600, 240, 1600, 2, "row"), ("alg_433_29", 1800, 360, 360, 2, "row"),
         ("laderman_class_333_23", 900, 900, 900, 2, "row")]
for name, P, Q, N, L, lay in cases:
    A, B = I.problem(P, Q, N, seed=3)
    def dev(x):
        if lay == "row":
            return torch.from_numpy(np.ascontiguousarray(x)).cuda()
        return torch.from_numpy(np.ascontiguousarray(x.T)).cuda().t()
    alg = F.load_alg(name)
    res = {}
    for fuse in (True, False):
        p = F.Plan(alg, P, Q, N, L, layout=lay, cse=False, fuse=fuse, collapse=False)
        C = p.execute(dev(A), dev(B))
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(3):
            p.execute(dev(A), dev(B), C)
        torch.cuda.synchronize()
        res[fuse] = (C.cpu().numpy(), p.stats()["launches"], (time.time() - t0) / 3)
    ref = O.fast(A, B, O.load_alg(F.alg_path(name)), L)
    nrm = np.linalg.norm(A) * np.linalg.norm(B)
    same = np.array_equal(res[True][0], res[False][0])
    err = np.max(np.abs(res[True][0] - ref)) / nrm
    print(f"{name} {P}x{Q}x{N} L={L} {lay}: fused==unfused {same}  err/nrm {err:.2e}  launches {res[True][1]:.0f} vs {res[False][1]:.0f}", flush=True)
    assert err < 1e-12
print("fused_check ok")
