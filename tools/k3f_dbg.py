import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import fmm_inputs as I
import paper_1409_2908_b200 as F
print("plan", flush=True)
p = F.Plan(F.load_alg("strassen_222_7"), 256, 256, 256, 1, fuse_output=True)
print("stats", p.stats()["fused_output"], flush=True)
A, B = I.problem(256, 256, 256, seed=51, kind="integers")
a = torch.from_numpy(A).cuda(); b = torch.from_numpy(B).cuda()
print("execute", flush=True)
C = p.execute(a, b)
print("sync", flush=True)
torch.cuda.synchronize()
print("ok", np.array_equal(C.cpu().numpy(), A @ B), flush=True)
