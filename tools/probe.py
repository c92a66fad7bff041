"""Quick GPU timing probe (development tool): library DGEMM vs cuBLAS, and fmm phases on a config."""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_1409_2908_b200 as F

def tm(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best

g = torch.Generator(device="cuda"); g.manual_seed(0)
for n in (2048, 4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g); b = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g)
    c = torch.empty_like(a)
    ms = tm(lambda: F.dgemm(a, b, c)); ms2 = tm(lambda: torch.matmul(a, b))
    print(json.dumps({"dgemm_n": n, "fmm_tflops": 2*n**3/ms/1e9, "cublas_tflops": 2*n**3/ms2/1e9}))
cfgs = [("winograd_class_222_7", 2, 8192, 8192, 8192, "col"), ("hk_class_323_15", 2, 12000, 1800, 12000, "row"),
        ("alg_424_26", 2, 16000, 2400, 16000, "row"), ("alg_433_29", 2, 18000, 3600, 3600, "row"),
        ("laderman_class_333_23", 2, 18000, 18000, 18000, "row")]
for name, L, P, Q, N, lay in cfgs:
    alg = F.load_alg(name)
    t0 = time.time(); p = F.Plan(alg, P, Q, N, L, layout=lay); tplan = time.time() - t0
    if lay == "row":
        A = torch.rand(P, Q, dtype=torch.float64, device="cuda", generator=g); B = torch.rand(Q, N, dtype=torch.float64, device="cuda", generator=g)
    else:
        A = torch.rand(Q, P, dtype=torch.float64, device="cuda", generator=g).t(); B = torch.rand(N, Q, dtype=torch.float64, device="cuda", generator=g).t()
    C = p.new_output()
    p.execute(A, B, C); torch.cuda.synchronize()
    best = None
    for _ in range(3):
        _, ph = p.execute_timed(A, B, C)
        if best is None or ph["total_ms"] < best["total_ms"]: best = ph
    st = p.stats()
    ms_cub = tm(lambda: torch.matmul(A, B), reps=2)
    print(json.dumps({"cfg": name, "P": P, "Q": Q, "N": N, "plan_s": tplan, **best,
                      "eff_tflops": 2*P*Q*N/best["total_ms"]/1e9, "cublas_tflops": 2*P*Q*N/ms_cub/1e9,
                      "gemm_tflops": st["gemm_flops"]/best["gemm_ms"]/1e9,
                      "add_GBs": st["add_bytes"]/(best["formation_ms"]+best["assembly_ms"])/1e6,
                      "ws_GB": p.workspace_bytes/1e9, **st}))
    del A, B, C, p; torch.cuda.empty_cache()
