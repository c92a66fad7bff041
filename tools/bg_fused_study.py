"""Fused leaf level in background mode (fuse_leaf_level = 2) against the default plan and the
addition-CTA fused mode (development tool): per BASELINE config, median execute time (CUDA events,
plain launches) and the max |difference| of C against the default plan's C.

  python tools/bg_fused_study.py [c2,c3,c4,c5t] [modes, e.g. default,1,2]
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
modes = (sys.argv[2] if len(sys.argv) > 2 else "default,2").split(",")
reps = int(os.environ.get("REPS", "7"))
for c in cfgs:
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
    ref = None
    for m in modes:
        fuse = {"default": False, "0": False, "1": True, "2": 2}[m]
        p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"], fuse=fuse, cuda_graphs=False)
        C = p.new_output()
        for _ in range(2):
            p.execute(A, B, C)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            p.execute(A, B, C)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        st = p.stats()
        if ref is None:
            ref = C.clone()
            diff = 0.0
        else:
            diff = (C - ref).abs().max().item()
        prof = {}
        try:
            for kind, lvl, t in p.execute_profile(A, B, C):
                prof[f"{kind}@{lvl}"] = round(prof.get(f"{kind}@{lvl}", 0.0) + t, 4)
        except Exception as e:  # noqa: BLE001
            prof = {"error": str(e)}
        print(json.dumps({"cfg": c, "mode": m, "ms": ms, "gflops": 2.0 * P * Q * N / ms / 1e6,
                          "fused_launches": st["fused_launches"], "collapsed": st["collapsed"],
                          "max_abs_diff_vs_first": diff, "profile_ms": prof}), flush=True)
        del p, C
        torch.cuda.empty_cache()
    del A, B, ref
    torch.cuda.empty_cache()
