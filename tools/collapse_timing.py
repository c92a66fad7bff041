"""Collapsed vs one-level-per-launch on BASELINE workloads: ms per execute (CUDA events) and the
plans' addition bytes."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1409_2908_b200 as F

for cfg in sys.argv[1:]:
    w = bench.WORKLOADS[cfg]
    A_np, B_np = bench.gen_inputs(w)
    A = bench.to_device(A_np, w["layout"], "cuda"); B = bench.to_device(B_np, w["layout"], "cuda")
    out = []
    for col in (False, True):
        p = F.Plan(F.load_alg(w["alg"]), w["P"], w["Q"], w["N"], w["L"], layout=w["layout"], collapse=col)
        C = p.new_output()
        for _ in range(2):
            p.execute(A, B, C)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            p.execute(A, B, C)
        e1.record(); torch.cuda.synchronize()
        st = p.stats()
        out.append(f"collapse={col}({int(st['collapsed'])}) {e0.elapsed_time(e1)/5:.2f} ms add {st['add_bytes']/1e9:.2f} GB launches {st['launches']:.0f}")
        del p, C
    print(cfg, " | ".join(out), flush=True)
    del A, B; torch.cuda.empty_cache()
