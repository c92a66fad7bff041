"""Background-bandwidth probe (development tool, timing only): with the library built with
-DFMM_BG_PROBE (FMM_BUILD_VARIANT=bg FMM_EXTRA_FLAGS=-DFMM_BG_PROBE python paper_1409_2908_b200/build.py,
then FMM_LIB_PATH=.../libfmm_bg.so), the plain leaf GEMM's idle producer warps 1-3 stream-copy
FMM_BG_BYTES bytes (read + write) of a separate buffer during each leaf GEMM launch; this prints the
median leaf-GEMM time per volume (profiles/r2_bg_probe.jsonl).

  BG_CFGS=c2,c4 BG_LIST=0,8,16,32,64 python tools/bg_probe.py
"""
import json, os, sys
import torch
sys.path.insert(0, "/root/repo")
import bench
import paper_1409_2908_b200 as F
for c in os.environ.get("BG_CFGS", "c2,c4").split(","):
    w = bench.WORKLOADS[c]
    P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
    g = torch.Generator(device="cuda"); g.manual_seed(0)
    if w["layout"] == "row":
        A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g); B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g)
    else:
        A = torch.rand(Q, P, dtype=torch.float64, device="cuda", generator=g).t(); B = torch.rand(N, Q, dtype=torch.float64, device="cuda", generator=g).t()
    for gb in [float(x) for x in os.environ.get("BG_LIST", "0,1,2,4,8,16").split(",")]:
        os.environ["FMM_BG_BYTES"] = str(int(gb * 1e9))
        p = F.Plan(F.load_alg(w["alg"]), P, Q, N, L, layout=w["layout"], cuda_graphs=False)
        C = p.new_output()
        p.execute(A, B, C); torch.cuda.synchronize()
        ts = sorted(p.execute_timed(A, B, C)[1]["gemm_ms"] for _ in range(5))
        print(json.dumps({"cfg": c, "bg_GB_copied": gb / 2, "bg_bytes_moved_GB": gb, "gemm_ms": ts[2]}), flush=True)
        del p, C; torch.cuda.empty_cache()
