"""Ramp-up curves on B200 (the paper's performance-vs-N figures):
effective TFLOP/s (2PQN/t) against N for the paper's three shape families -- square N x N x N,
"outer product" N x 1600 x N and tall-skinny N x 2400 x 2400 -- for cuBLAS DGEMM, this
library's classical DMMA GEMM (L = 0), each fast algorithm at its best L in {1, 2, 3} ("best of L",
as the paper reports), and the selector's choice (fmm_select, cost model only).
One JSON line per (family, N).  Usage: python tools/ramp_study.py [family ...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fmm_inputs as I  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

FAMILIES = {
    "square": [(n, n, n) for n in (1024, 2048, 3072, 4096, 6144, 8192, 12288)],
    "outer": [(n, 1600, n) for n in (2048, 4096, 8192, 12288, 16384)],
    "tall": [(n, 2400, 2400) for n in (4800, 9600, 19200, 38400)],
}
ALGS = ["winograd_class_222_7", "hk_class_323_15", "alg_424_26", "laderman_class_333_23", "alg_433_29",
        "flip_234_20"]


def timed(fn, reps=3):
    fn()  # builds the plan's launch tables
    fn()  # captures the CUDA graph (cuda_graphs option); later calls replay it
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def plan_ms(alg, P, Q, N, L, A, B):
    try:
        p = F.Plan(alg, P, Q, N, L)
    except F.FmmError as e:
        return None, str(e)[:60]
    C = p.new_output()
    ms = timed(lambda: p.execute(A, B, C))
    del p, C
    return ms, None


def main():
    fams = sys.argv[1:] or list(FAMILIES)
    algs = [F.load_alg(n) for n in ALGS]
    every = [F.load_alg(n[:-4]) for n in sorted(os.listdir(os.path.join(ROOT, "algs"))) if n.endswith(".txt")]
    for fam in fams:
        for (P, Q, N) in FAMILIES[fam]:
            A_np, B_np = I.problem(P, Q, N, seed=0)
            A, B = torch.from_numpy(A_np).cuda(), torch.from_numpy(B_np).cuda()
            del A_np, B_np
            fl = 2.0 * P * Q * N
            tf = lambda ms: fl / (ms * 1e-3) / 1e12 if ms else None  # noqa: E731
            row = {"family": fam, "shape": [P, Q, N]}
            row["cublas"] = tf(timed(lambda: torch.matmul(A, B)))
            ms, _ = plan_ms(algs[0], P, Q, N, 0, A, B)
            row["dmma_classical"] = tf(ms)
            best = {}
            for a, name in zip(algs, ALGS):
                cands = []
                for L in (1, 2, 3):
                    ms, err = plan_ms(a, P, Q, N, L, A, B)
                    if ms:
                        cands.append((ms, L))
                if cands:
                    ms, L = min(cands)
                    best[name] = {"L": L, "tflops": tf(ms)}
            row["fast_best_of_L"] = best
            sel, Ls, pms = F.select(every, P, Q, N, 3, "row")
            if sel is not None:
                ms, err = plan_ms(sel, P, Q, N, Ls, A, B)
                row["select"] = {"plan": sel.name, "L": Ls, "predicted_ms": pms, "ms": ms, "tflops": tf(ms)}
            print(json.dumps(row), flush=True)
            del A, B
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
