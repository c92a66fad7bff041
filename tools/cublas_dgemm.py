"""cuBLAS DGEMM (torch.matmul float64) and fp64 copy rates on this box: the classical baseline
and the HBM denominator for the fp64 path. Prints one JSON line per measurement."""
import json, time, torch

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

dev = torch.device("cuda")
g = torch.Generator(device=dev); g.manual_seed(0)
for n in (2048, 4096, 8192):
    a = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    b = torch.rand(n, n, dtype=torch.float64, device=dev, generator=g) * 2 - 1
    ms = t(lambda: torch.matmul(a, b))
    print(json.dumps({"what": "cublas_dgemm", "n": n, "ms": ms, "tflops": 2 * n**3 / ms / 1e9}))
for (bt, m, k, n) in ((49, 2048, 2048, 2048), (676, 1000, 600, 1000), (841, 1125, 400, 400)):
    a = torch.rand(bt, m, k, dtype=torch.float64, device=dev, generator=g)
    b = torch.rand(bt, k, n, dtype=torch.float64, device=dev, generator=g)
    ms = t(lambda: torch.bmm(a, b), reps=3)
    print(json.dumps({"what": "cublas_bmm", "shape": [bt, m, k, n], "ms": ms, "tflops": 2 * bt * m * k * n / ms / 1e9}))
    del a, b
x = torch.empty(2**28, dtype=torch.float64, device=dev); y = torch.empty_like(x)
ms = t(lambda: y.copy_(x), reps=10)
print(json.dumps({"what": "copy_f64", "bytes": 2 * x.numel() * 8, "ms": ms, "gbs": 2 * x.numel() * 8 / ms / 1e6}))
