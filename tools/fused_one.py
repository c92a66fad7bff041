"""One fused execute of a given case (for compute-sanitizer): alg P Q N L [layout]."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fmm_inputs as I  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

name, P, Q, N, L = sys.argv[1], *map(int, sys.argv[2:6])
A, B = I.problem(P, Q, N, seed=3)
p = F.Plan(F.load_alg(name), P, Q, N, L, cse=False)
C = p.execute(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
torch.cuda.synchronize()
print("ok", float(np.abs(C.cpu().numpy() - A @ B).max()))
