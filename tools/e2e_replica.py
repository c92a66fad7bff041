"""Replica of fmm_execute_host_async's two-set pipeline with torch streams and events, to see where
the e2e step time goes (c2)."""
import json, sys
import torch
sys.path.insert(0, ".")
import paper_1409_2908_b200 as F

n = 8192
plan = F.Plan(F.load_alg("winograd_class_222_7"), n, n, n, 2, layout="col")
Ah = torch.empty(n, n, dtype=torch.float64).pin_memory(); Ah.uniform_(-1, 1)
Bh = torch.empty(n, n, dtype=torch.float64).pin_memory(); Bh.uniform_(-1, 1)
Ch = torch.empty(n, n, dtype=torch.float64).pin_memory()
sets = [[torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(3)] for _ in range(2)]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)
K = 8
marks = []
ev_comp = [None, None]; ev_out = [None, None]
t0 = ev(); t0.record(s_c)
for i in range(K):
    b = i % 2
    A, B, C = sets[b]
    m = [ev() for _ in range(6)]
    if ev_comp[b] is not None: s_in.wait_event(ev_comp[b])
    m[0].record(s_in)
    with torch.cuda.stream(s_in):
        A.copy_(Ah, non_blocking=True); B.copy_(Bh, non_blocking=True)
    m[1].record(s_in)
    s_c.wait_event(m[1])
    if ev_out[b] is not None: s_c.wait_event(ev_out[b])
    m[2].record(s_c)
    plan.execute(A.t(), B.t(), C.t(), stream=s_c)
    m[3].record(s_c)
    ev_comp[b] = m[3]
    s_out.wait_event(m[3])
    m[4].record(s_out)
    with torch.cuda.stream(s_out):
        Ch.copy_(C, non_blocking=True)
    m[5].record(s_out)
    ev_out[b] = m[5]
    marks.append(m)
torch.cuda.synchronize()
for i, m in enumerate(marks):
    v = [t0.elapsed_time(x) for x in m]
    print(f"step {i}: in {v[0]:.1f}-{v[1]:.1f}  compute {v[2]:.1f}-{v[3]:.1f}  out {v[4]:.1f}-{v[5]:.1f}")
print(json.dumps({"ms_per_step_steady": (t0.elapsed_time(marks[-1][5]) - t0.elapsed_time(marks[1][5])) / (K - 2)}))
