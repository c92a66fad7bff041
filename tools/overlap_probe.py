"""Does host<->device traffic slow the fast multiplication down?  Time plan.execute on its stream
alone and with an H2D + D2H copy loop running on two other streams (c2 workload)."""
import json, sys, time
import torch
sys.path.insert(0, ".")
import bench
import paper_1409_2908_b200 as F

w = bench.WORKLOADS["c2"]
A_np, B_np = bench.gen_inputs(w)
A = bench.to_device(A_np, "col", "cuda"); B = bench.to_device(B_np, "col", "cuda")
plan = F.Plan(F.load_alg(w["alg"]), 8192, 8192, 8192, 2, layout="col")
C = plan.new_output()
n = 8192
Ah = torch.empty(2 * n, n, dtype=torch.float64).pin_memory()
Ch = torch.empty(n, n, dtype=torch.float64).pin_memory()
Ad = torch.empty(2 * n, n, dtype=torch.float64, device="cuda"); Cd = torch.empty(n, n, dtype=torch.float64, device="cuda")
s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def compute(k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    for _ in range(k):
        plan.execute(A, B, C, stream=s0)
    e1.record(s0)
    return e0, e1
for _ in range(3):
    plan.execute(A, B, C, stream=s0)
torch.cuda.synchronize()
e0, e1 = compute(6); torch.cuda.synchronize()
alone = e0.elapsed_time(e1) / 6
# with copies
c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
c0.record(s1)
for _ in range(8):
    with torch.cuda.stream(s1): Ad.copy_(Ah, non_blocking=True)
    with torch.cuda.stream(s2): Ch.copy_(Cd, non_blocking=True)
c1.record(s1)
e0, e1 = compute(6)
torch.cuda.synchronize()
print(json.dumps({"compute_alone_ms": alone, "compute_with_copies_ms": e0.elapsed_time(e1) / 6,
                  "h2d_loop_GBs": 8 * Ah.numel() * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9}))
