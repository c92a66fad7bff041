"""Per-launch times of one BASELINE config's step (fmm_execute_profile; development tool):
  python tools/launch_profile.py c4 [reps]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

c = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
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
p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"])
C = p.new_output()
p.execute(A, B, C)
runs = [p.execute_profile(A, B, C) for _ in range(reps)]
for q, (kind, level, _) in enumerate(runs[0]):
    ms = sorted(r[q][2] for r in runs)[len(runs) // 2]
    print(json.dumps({"cfg": c, "launch": q, "kind": kind, "level": level, "ms": ms}))
