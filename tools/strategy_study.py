"""Strategy x CSE study on B200 (the paper's Fig. 2 question):
pairwise (daxpy chains) vs write-once vs streaming addition kernels, CSE on / off (streaming keeps
the common subexpressions in registers; write-once and pairwise write them to memory once per
node), for <4,2,4;26> on N x 1600 x N (the paper's outer-product
family), <4,2,3;20> on N x N x N (Fig. 2's second panel; the <2,3,4;20> of algs/ under Prop. 2) and
the c2 / c4 workloads.  One JSON line per (workload, strategy, cse)."""
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

WL = [("alg_424_26", 8000, 1600, 8000, 2, "row"), ("alg_424_26", 16000, 1600, 16000, 2, "row"),
      ("winograd_class_222_7", 8192, 8192, 8192, 2, "col"), ("alg_424_26", 16000, 2400, 16000, 2, "row"),
      ("laderman_class_333_23", 9000, 9000, 9000, 2, "row"), ("flip_234_20^NMK", 7200, 7200, 7200, 2, "row")]


def load(name):
    base, _, perm = name.partition("^")
    alg = F.load_alg(base)
    if perm:
        alg = alg.permute(F.Algorithm.PERMS.index(perm))
    return alg


for name, P, Q, N, L, lay in WL:
    A_np, B_np = I.problem(P, Q, N, seed=0, layout=lay)
    A = bench.to_device(A_np, lay, "cuda")
    B = bench.to_device(B_np, lay, "cuda")
    for strategy in ("streaming", "write_once", "pairwise"):
        for cse in (False, True):
            p = F.Plan(load(name), P, Q, N, L, layout=lay, strategy=strategy, cse=cse)
            st = p.stats()
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
            add_ms = ph[0] + ph[2]
            print(json.dumps({"alg": name, "shape": [P, Q, N], "L": L, "layout": lay, "strategy": strategy, "cse": cse,
                              "ms": float(ph[3]), "tflops": 2.0 * P * Q * N / (ph[3] * 1e-3) / 1e12,
                              "formation_ms": float(ph[0]), "gemm_ms": float(ph[1]), "assembly_ms": float(ph[2]),
                              "add_bytes": st["add_bytes"], "add_flops": st["add_flops"], "collapsed": st["collapsed"],
                              "launches": st["launches"],
                              "add_gbs": st["add_bytes"] / (add_ms * 1e-3) / 1e9}), flush=True)
            del p, C
    del A, B
    torch.cuda.empty_cache()
