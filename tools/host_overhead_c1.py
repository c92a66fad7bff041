"""Host overhead per call of fmm_execute and torch.matmul on c1, and cuBLAS replayed from a CUDA graph
(development tool for the small-path study)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_1409_2908_b200 as F
A = torch.rand(256, 256, dtype=torch.float64, device="cuda"); B = torch.rand(256, 256, dtype=torch.float64, device="cuda")
p = F.Plan(F.load_alg("strassen_222_7"), 256, 256, 256, 1)
C = p.new_output()
s = torch.cuda.current_stream()
for _ in range(20): p.execute(A, B, C, stream=s)
torch.cuda.synchronize()
for name, fn in [("fmm", lambda: p.execute(A, B, C, stream=s)), ("cublas", lambda: torch.matmul(A, B, out=C))]:
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(2000): fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        print(name, "host us/call %.2f" % ((t1 - t0) / 2000 * 1e6), "total us/call %.2f" % ((t2 - t0) / 2000 * 1e6))
# graph-captured cuBLAS: device-bound time
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(20): torch.matmul(A, B, out=C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50): g.replay()
e1.record(); torch.cuda.synchronize()
print("cublas in a CUDA graph: us per matmul %.2f" % (e0.elapsed_time(e1) / 1000 * 1e3))
