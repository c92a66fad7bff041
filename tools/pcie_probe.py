"""PCIe / e2e probe: H2D, D2H, both at once, blocking and pipelined host execution (c2)."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1409_2908_b200 as F

n = 8192
Ah = torch.empty(n, n, dtype=torch.float64).pin_memory(); Ah.uniform_(-1, 1)
Bh = torch.empty(n, n, dtype=torch.float64).pin_memory(); Bh.uniform_(-1, 1)
Ch = torch.empty(n, n, dtype=torch.float64).pin_memory()
Ad = torch.empty(n, n, dtype=torch.float64, device="cuda"); Cd = torch.empty_like(Ad)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def wall(fn, reps=3):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / reps * 1e3
b = n * n * 8
print(json.dumps({"h2d_GBs": b / wall(lambda: Ad.copy_(Ah, non_blocking=True)) / 1e6}))
print(json.dumps({"d2h_GBs": b / wall(lambda: Ch.copy_(Cd, non_blocking=True)) / 1e6}))
def both():
    with torch.cuda.stream(s1): Ad.copy_(Ah, non_blocking=True)
    with torch.cuda.stream(s2): Ch.copy_(Cd, non_blocking=True)
print(json.dumps({"both_ms": wall(both), "one_way_ms": b / 1e6 / 55}))
plan = F.Plan(F.load_alg("winograd_class_222_7"), n, n, n, 2, layout="col")
At, Bt, Ct = Ah.t(), Bh.t(), Ch.t()
print(json.dumps({"blocking_ms": wall(lambda: plan.execute_host(At, Bt, Ct))}))
def pipe(k=6):
    for _ in range(k): plan.execute_host(At, Bt, Ct, asynchronous=True)
    plan.sync()
print(json.dumps({"pipelined_ms_per_step": wall(pipe, reps=2) / 6}))
s_user = torch.cuda.Stream()
def pipe_stream(k=6):
    for _ in range(k): plan.execute_host(At, Bt, Ct, asynchronous=True, stream=s_user)
    plan.sync()
print(json.dumps({"pipelined_ms_per_step_user_stream": wall(pipe_stream, reps=2) / 6}))
