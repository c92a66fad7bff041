"""One traced execute of the fused leaf level (FMM_FUSE_DEBUG=trace prints per-CTA timelines)."""
import os
import sys

import torch

os.environ["FMM_FUSE_DEBUG"] = "trace"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1409_2908_b200 as F  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c5t"]
A_np, B_np = bench.gen_inputs(w)
A = bench.to_device(A_np, w["layout"], "cuda")
B = bench.to_device(B_np, w["layout"], "cuda")
p = F.Plan(F.load_alg(w["alg"]), w["P"], w["Q"], w["N"], w["L"], layout=w["layout"])
C = p.execute(A, B)
torch.cuda.synchronize()
print("---- second run ----", flush=True)
p.execute(A, B, C)
torch.cuda.synchronize()
