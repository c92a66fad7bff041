"""c1 (Strassen L=1, 256^3): per-launch times and the whole step (graph replay) against cuBLAS,
for the small-problem path study (development tool):  python tools/c1_study.py [workload]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

c = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = bench.WORKLOADS[c]
P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
g = torch.Generator(device="cuda")
g.manual_seed(0)
A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout="row")
C = p.new_output()
p.execute(A, B, C)
runs = [p.execute_profile(A, B, C) for _ in range(7)]
for q, (kind, level, _) in enumerate(runs[0]):
    ms = sorted(r[q][2] for r in runs)[len(runs) // 2]
    print(json.dumps({"cfg": c, "launch": q, "kind": kind, "level": level, "ms": ms}))


def timeit(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_fmm = timeit(lambda: p.execute(A, B, C))
t_cub = timeit(lambda: torch.matmul(A, B))
err = (C - A @ B).abs().max().item()
print(json.dumps({"cfg": c, "step_ms": t_fmm, "cublas_ms": t_cub, "vs_cublas": t_cub / t_fmm, "max_err": err,
                  "stats": p.stats()}))

# the classical product below the cutoff (L = 0) through the same one launch
p0 = F.Plan(F.load_alg(w["alg"]), P, Q, N, 0, layout="row")
C0 = p0.new_output()
t0 = timeit(lambda: p0.execute(A, B, C0))
g = torch.cuda.CUDAGraph()
Cg = torch.empty_like(C)
with torch.cuda.graph(g):
    for _ in range(20):
        torch.matmul(A, B, out=Cg)
torch.cuda.synchronize()
t_cub_graph = timeit(lambda: g.replay(), reps=50) / 20
print(json.dumps({"cfg": c, "L0_step_ms": t0, "L0_stats_small": p0.stats()["small_fused"], "cublas_graph_ms": t_cub_graph,
                  "cublas_plain_out_ms": timeit(lambda: torch.matmul(A, B, out=Cg)),
                  "max_err_L0": (C0 - A @ B).abs().max().item()}))
