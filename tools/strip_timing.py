"""Peel-strip timing (development tool): median strips_ms / total_ms of fmm_execute_timed for the
configs that peel (c3 by default), and an element-wise check of C against the library's own
classical DMMA GEMM (L = 0) on the same inputs.

  python tools/strip_timing.py [c3,...]     (FMM_SKINNY_ROWS=narrow: the 32-column row-strip form)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

cfgs = (sys.argv[1] if len(sys.argv) > 1 else "c3").split(",")
reps = int(os.environ.get("REPS", "11"))
g = torch.Generator(device="cuda")
g.manual_seed(0)
for c in cfgs:
    w = bench.WORKLOADS[c]
    P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
    if w["layout"] == "row":
        A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    else:
        A = (torch.rand(Q, P, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
        B = (torch.rand(N, Q, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t()
    p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"])
    C = p.new_output()
    for _ in range(2):
        p.execute(A, B, C)
    torch.cuda.synchronize()
    ts = [p.execute_timed(A, B, C)[1] for _ in range(reps)]
    med = lambda key: sorted(t[key] for t in ts)[len(ts) // 2]  # noqa: E731
    ref = F.Plan(F.load_alg(w["alg"]), P, Q, N, 0, layout=w["layout"]).execute(A, B)
    torch.cuda.synchronize()
    err = (C - ref).abs().max().item()
    print(json.dumps({"cfg": c, "rows_form": os.environ.get("FMM_SKINNY_ROWS", "wide"), "strips_ms": med("strips_ms"),
                      "total_ms": med("total_ms"), "gemm_ms": med("gemm_ms"), "max_err_vs_classical": err,
                      "bound": 1e-10 * (A.norm() * B.norm()).item()}), flush=True)
    del p, C, ref, A, B
    torch.cuda.empty_cache()
