"""Per-phase device times of one plan (formation / leaf products / assembly + strips), for checking
the cost model (fmm_plan_predict) phase by phase.  Usage: phase_probe.py ALG P Q N L [layout]."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import fmm_inputs as I  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402


def main():
    name, P, Q, N, L = sys.argv[1], *map(int, sys.argv[2:6])
    lay = sys.argv[6] if len(sys.argv) > 6 else "row"
    base, _, perm = name.partition("^")
    alg = F.load_alg(base)
    if perm:
        alg = alg.permute(F.Algorithm.PERMS.index(perm))
    A_np, B_np = I.problem(P, Q, N, seed=0, layout=lay)
    A, B = bench.to_device(A_np, lay, "cuda"), bench.to_device(B_np, lay, "cuda")
    p = F.Plan(alg, P, Q, N, L, layout=lay)
    C = p.new_output()
    for _ in range(2):
        p.execute(A, B, C)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(5)]
    for e in (x for r in evs for x in r):
        e.record()
    torch.cuda.synchronize()
    for k in range(5):
        p.execute_events(A, B, C, evs[k])
    torch.cuda.synchronize()
    ph = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[0].elapsed_time(e[3])]
                   for e in evs]).mean(axis=0)
    st = p.stats()
    print(json.dumps({"alg": name, "shape": [P, Q, N], "L": L, "layout": lay, "formation_ms": ph[0], "gemm_ms": ph[1],
                      "assembly_ms": ph[2], "total_ms": ph[3], "pred_ms": alg.predict_ms(P, Q, N, L, lay),
                      "stats": st}), flush=True)


if __name__ == "__main__":
    main()
