"""Cutoff / shape-matching study: for each BASELINE shape, measure the
configured algorithm at L = 0..3, the selector's choice (fmm_select over every algorithm file and
its Prop. 1/2 permutations) and report them next to the cost model's predictions.
Writes one JSON object per line to stdout."""
import glob
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402


def time_plan(alg, w, L, A, B, reps=3):
    try:
        p = F.Plan(alg, w["P"], w["Q"], w["N"], L, layout=w["layout"])
    except F.FmmError as e:
        return None, str(e)[:80]
    try:
        C = p.new_output()
    except torch.OutOfMemoryError as e:  # the plan's workspace left no room for C (c5 at L = 3)
        del p
        torch.cuda.empty_cache()
        return None, "out of memory: " + str(e)[:60]
    p.execute(A, B, C)  # builds the launch tables
    p.execute(A, B, C)  # captures the CUDA graph; the timed calls replay it
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        p.execute(A, B, C)
    e1.record()
    torch.cuda.synchronize()
    del p, C
    torch.cuda.empty_cache()
    return e0.elapsed_time(e1) / reps, None


def main():
    names = [os.path.basename(p)[:-4] for p in sorted(glob.glob(os.path.join(ROOT, "algs", "*.txt")))]
    algs = [F.load_alg(n) for n in names]
    cfgs = sys.argv[1:] or ["c2", "c3", "c4", "c5t", "c1"]
    for cfg in cfgs:
        w = bench.WORKLOADS[cfg]
        A_np, B_np = bench.gen_inputs(w)
        A = bench.to_device(A_np, w["layout"], "cuda")
        B = bench.to_device(B_np, w["layout"], "cuda")
        flops = 2.0 * w["P"] * w["Q"] * w["N"]
        base = F.load_alg(w["alg"])
        rows = []
        for L in range(0, 4):
            pred = base.predict_ms(w["P"], w["Q"], w["N"], L, w["layout"])
            ms, err = time_plan(base, w, L, A, B)
            rows.append({"alg": w["alg"], "L": L, "pred_ms": pred, "ms": ms, "tflops": flops / (ms * 1e-3) / 1e12 if ms else None,
                         "err": err})
        sel, Ls, pms = F.select(algs, w["P"], w["Q"], w["N"], 3, w["layout"])
        if sel is not None:
            ms, err = time_plan(sel, w, Ls, A, B)
            rows.append({"alg": "select:" + sel.name, "L": Ls, "pred_ms": pms, "ms": ms,
                         "tflops": flops / (ms * 1e-3) / 1e12 if ms else None, "err": err})
        print(json.dumps({"workload": cfg, "shape": [w["P"], w["Q"], w["N"]], "layout": w["layout"], "rows": rows}), flush=True)
        del A, B
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
