"""Leaf-GEMM study (development tool): for each BASELINE config, the leaf products' time and
fraction of the DMMA peak from fmm_execute_timed (per-launch events), for the chooser's tile width
and for forced widths (FMM_GEMM_BN).  Inputs are device-generated (timing does not depend on values).

  python tools/leaf_gemm_study.py [c2,c3,c4,c5t] [bn list, e.g. auto,128,112,96,80]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

cfgs = (sys.argv[1] if len(sys.argv) > 1 else "c2,c3,c4,c5t").split(",")
bns = (sys.argv[2] if len(sys.argv) > 2 else "auto").split(",")
reps = int(os.environ.get("REPS", "5"))
peak, _ = F.probe_fp64_peak()
g = torch.Generator(device="cuda")
g.manual_seed(0)
for c in cfgs:
    w = bench.WORKLOADS[c]
    P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
    if w["layout"] == "row":
        A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g)
        B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g)
    else:
        A = torch.rand(Q, P, dtype=torch.float64, device="cuda", generator=g).t()
        B = torch.rand(N, Q, dtype=torch.float64, device="cuda", generator=g).t()
    for bn in bns:
        if bn == "auto":
            os.environ.pop("FMM_GEMM_BN", None)
        else:
            os.environ["FMM_GEMM_BN"] = bn
        p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"])
        C = p.new_output()
        for _ in range(2):
            p.execute(A, B, C)
        torch.cuda.synchronize()
        ts = [p.execute_timed(A, B, C)[1] for _ in range(reps)]
        gm = sorted(t["gemm_ms"] for t in ts)[len(ts) // 2]
        tot = sorted(t["total_ms"] for t in ts)[len(ts) // 2]
        st = p.stats()
        print(json.dumps({"cfg": c, "bn": bn, "gemm_ms": gm, "total_ms": tot, "leaf_tflops": st["leaf_flops"] / gm / 1e9,
                          "frac": st["leaf_flops"] / gm / 1e9 / peak, "peak": peak,
                          "eff_tflops": 2.0 * P * Q * N / tot / 1e9}), flush=True)
        del p, C
        torch.cuda.empty_cache()
    del A, B
    torch.cuda.empty_cache()
os.environ.pop("FMM_GEMM_BN", None)
