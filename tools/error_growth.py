"""Error growth of the GPU fast product against L (reported, not gated):
e_L = max |C_gpu,L - C_exact| / (||A||_F ||B||_F) for L = 0..3 on uniform[-1,1] inputs, with C_exact
the product in 80-bit extended precision (numpy longdouble), next to the bound derived from (U,V,W)
(oracle.error_bound) and the oracle's own fast result at the same L.

  python tools/error_growth.py > profiles/r2_error_growth.jsonl
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fmm_inputs as I  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = [("strassen_222_7", 512, 512, 512), ("winograd_class_222_7", 512, 512, 512),
         ("hk_class_323_15", 540, 216, 540), ("alg_424_26", 512, 128, 512), ("laderman_class_333_23", 540, 540, 540)]
for name, P, Q, N in CASES:
    A, B = I.problem(P, Q, N, seed=5)
    exact = np.matmul(A.astype(np.longdouble), B.astype(np.longdouble))
    nrm = float(np.linalg.norm(A) * np.linalg.norm(B))
    oa = O.load_alg(F.alg_path(name))
    for L in range(4):
        p = F.Plan(F.load_alg(name), P, Q, N, L)
        used = int(p.stats()["levels"])
        if used < L:
            break
        C = p.execute(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
        eg = float(np.max(np.abs(C.astype(np.longdouble) - exact)))
        Co = O.fast(A, B, oa, L)
        eo = float(np.max(np.abs(Co.astype(np.longdouble) - exact)))
        try:
            bound = O.error_bound(oa, Q, L, float(np.abs(A).max()), float(np.abs(B).max()))
        except AssertionError:
            bound = None
        print(json.dumps({"alg": name, "shape": [P, Q, N], "L": L, "e_gpu": eg / nrm, "e_oracle": eo / nrm,
                          "max_abs_gpu": eg, "max_abs_oracle": eo, "bound_abs": bound,
                          "gpu_over_bound": (eg / bound) if bound else None,
                          "gpu_vs_oracle": float(np.max(np.abs(C - Co))) / nrm}), flush=True)
