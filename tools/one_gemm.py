"""Run one BASELINE config's plan a few times (development tool for ncu captures of the leaf GEMM):
  python tools/one_gemm.py c2 [reps]       (FMM_GEMM_BN forces the tile width)
Inputs are device-generated; the last execute is a plain, timed one (no CUDA graph)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

c = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = bench.WORKLOADS[c]
P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
g = torch.Generator(device="cuda")
g.manual_seed(0)
if w["layout"] == "row":
    A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g)
    B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g)
else:
    A = torch.rand(Q, P, dtype=torch.float64, device="cuda", generator=g).t()
    B = torch.rand(N, Q, dtype=torch.float64, device="cuda", generator=g).t()
p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"], cuda_graphs=False)
C = p.new_output()
for _ in range(reps):
    _, t = p.execute_timed(A, B, C)
print(c, os.environ.get("FMM_GEMM_BN", "auto"), t)
