"""Time one workload's execute with CUDA events (diagnostics for the fused leaf level)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = bench.WORKLOADS[cfg]
A_np, B_np = bench.gen_inputs(w)
A = bench.to_device(A_np, w["layout"], "cuda")
B = bench.to_device(B_np, w["layout"], "cuda")
fuse = os.environ.get("FMM_NO_FUSE", "0") != "1"
p = F.Plan(F.load_alg(w["alg"]), w["P"], w["Q"], w["N"], w["L"], layout=w["layout"], fuse=fuse, collapse=os.environ.get("FMM_NO_COLLAPSE", "0") != "1" and not fuse)
C = p.new_output()
for _ in range(3):
    p.execute(A, B, C)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 5
e0.record()
for _ in range(n):
    p.execute(A, B, C)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"{cfg} fuse={fuse} dbg={os.environ.get('FMM_FUSE_DEBUG', '-')} stages={os.environ.get('FMM_STAGES','-')}: "
      f"{ms:.2f} ms/step, {2*w['P']*w['Q']*w['N']/ms/1e9:.0f} GFLOPS, launches {p.stats()['launches']:.0f}", flush=True)
