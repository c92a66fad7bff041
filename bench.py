#!/usr/bin/env python
"""bench.py — effective FP64 GFLOPS (2MKN/t) of the recursive fast matrix multiplication hot path
(arXiv 1409.2908) on B200, through the repo's C-ABI library.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

One step = one fmm_execute of the whole hot path (S/T formation at every level, the grouped DMMA
leaf GEMM, C assembly at every level, peel strips) over one synthetic input pair already
resident in HBM; for N > 1 each rank computes its leaf shard and the partial C are summed with
one NCCL reduce, inside the timed region.  Prints ONE JSON line on rank 0.

Default workload = BASELINE.json configs[1] (c2): Strassen-Winograd-class <2,2,2;7>, L = 2,
8192 x 8192 x 8192, column-major, uniform[-1,1] from seeds 0/1.  The other configs are parity
cases (tests/) and can be selected with --workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective FP64 GFLOPS (2MKN/t) per <M,K,N;R> algorithm vs FP64 peak, 1/2/4/8 GPU"
WORKLOADS = {
    "c1": dict(alg="strassen_222_7", L=1, P=256, Q=256, N=256, layout="row",
               desc="Strassen <2,2,2;7>, L=1, 256x256x256"),
    "c2": dict(alg="winograd_class_222_7", L=2, P=8192, Q=8192, N=8192, layout="col",
               desc="Strassen-Winograd-class <2,2,2;7>, L=2, 8192x8192x8192, column-major"),
    "c3": dict(alg="hk_class_323_15", L=2, P=12000, Q=1800, N=12000, layout="row",
               desc="<3,2,3;15>, L=2, 12000x1800x12000 (peeled at level 2)"),
    "c4": dict(alg="alg_424_26", L=2, P=16000, Q=2400, N=16000, layout="row",
               desc="<4,2,4;26>, L=2, 16000x2400x16000"),
    "c5": dict(alg="laderman_class_333_23", L=2, P=18000, Q=18000, N=18000, layout="row",
               desc="<3,3,3;23>, L=2, 18000x18000x18000"),
    "c5t": dict(alg="alg_433_29", L=2, P=18000, Q=3600, N=3600, layout="row",
                desc="<4,3,3;29>, L=2, 18000x3600x3600"),
}
HBM_FALLBACK = 6650.0


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except OSError:
        return {"hbm_gbs": HBM_FALLBACK}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.rows, self.proc, self.th = [], None, None
        self.device = device

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        def rd():
            for ln in self.proc.stdout:
                self.rows.append([x.strip() for x in ln.split(",")])
        self.th = threading.Thread(target=rd, daemon=True)
        self.th.start()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def gen_inputs(w, seed=0):
    import fmm_inputs as I
    return I.problem(w["P"], w["Q"], w["N"], seed=seed, kind="uniform", layout=w["layout"])


def to_device(x, layout, device):
    import numpy as np
    import torch
    if layout == "row":
        return torch.from_numpy(np.ascontiguousarray(x)).to(device)
    return torch.from_numpy(np.ascontiguousarray(x.T)).to(device).t()


def cpu_model():
    """The host CPU's model name (/proc/cpuinfo), for the cpu_baseline record."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_sample(w, A, B, frac):
    """The oracle as it stands (oracle_fast, same algorithm and L) on the leading
    (frac P) x (frac Q) x (frac N) sub-problem of the workload's own A and B.  One run."""
    import numpy as np
    from oracle import oracle as O
    alg = O.load_alg(os.path.join(ROOT, "algs", w["alg"] + ".txt"))
    p, q, n = (max(1, int(w["P"] * frac)), max(1, int(w["Q"] * frac)), max(1, int(w["N"] * frac)))
    As, Bs = A[:p, :q], B[:q, :n]
    t0 = time.perf_counter()
    O.fast(As, Bs, alg, w["L"])
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    return {"value": 2.0 * p * q * n / dt / 1e9, "unit": "GFLOPS", "cores": cores, "kind": "oracle",
            "seconds": dt, "cpu_model": cpu_model(),
            "sample": f"oracle_fast ({w['alg']}, L={w['L']}) on the leading {p}x{q}x{n} sub-problem of the "
                      f"workload's A,B (one run, OpenMP over {cores} threads); value = 2pqn/t"}


def run_reference(args, w):
    """--impl reference: the oracle, as it stands, on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    A, B = gen_inputs(w)
    from oracle import oracle as O
    O.build()
    frac = args.ref_frac
    for _ in range(args.warmup):
        cpu_oracle_sample(w, A, B, frac)
    vals, secs = [], 0.0
    last = None
    for _ in range(args.steps):
        last = cpu_oracle_sample(w, A, B, frac)
        secs += last["seconds"]
        vals.append(last["value"])
    p, q, n = int(w["P"] * frac), int(w["Q"] * frac), int(w["N"] * frac)
    value = args.steps * 2.0 * p * q * n / secs / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w["desc"], "sample": last["sample"]},
            "cpu_baseline": {"value": value, "unit": "GFLOPS", "cores": last["cores"], "kind": "oracle",
                             "sample": last["sample"], "cpu_model": last["cpu_model"]},
            "e2e": {"value": value, "unit": "GFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--strategy", default="streaming", choices=["streaming", "write_once", "pairwise"])
    ap.add_argument("--cse", type=int, default=1)
    ap.add_argument("--cpu-frac", type=float, default=1.0, help="oracle sample size (fraction of each dim)")
    ap.add_argument("--ref-frac", type=float, default=0.25, help="reference-arm sample (fraction of each dim)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--fuse", type=int, default=0, help="fused leaf level (formation/GEMM/assembly in one launch)")
    ap.add_argument("--collapse", type=int, default=1, help="last two levels' formation / assembly in one pass each")
    ap.add_argument("--shard-mode", default="leaf", choices=["leaf", "top"],
                    help="N > 1: leaf-level HYBRID sharding or the top-level products in contiguous ranges")
    ap.add_argument("--combine", default="torch", choices=["torch", "lib", "p2p"],
                    help="N > 1: partial-C reduce by torch.distributed (NCCL) or inside fmm_execute (fmm_plan_create_dist)")
    ap.add_argument("--output", default="root", choices=["root", "slabs"],
                    help="N > 1: C summed onto rank 0, or slab-distributed (slab g of C summed onto rank g)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1: gloo only to exercise the multi-rank control flow where ranks share a GPU (not a measurement)")
    ap.add_argument("--no-other", action="store_true", help="skip timing the other leaf-level schedule (fused vs separate)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if args.dist_backend == "gloo":
            # control-flow check of the N > 1 path on a box with fewer GPUs than ranks (ranks share
            # devices; gloo carries the collectives): its numbers are not measurements
            local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    device = torch.device(f"cuda:{torch.cuda.current_device()}")
    import __graft_entry__
    __graft_entry__.build()
    import paper_1409_2908_b200 as F
    from paper_1409_2908_b200.dist import combine_partials, scatter_partials

    P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
    A_np, B_np = gen_inputs(w)
    A = to_device(A_np, w["layout"], device)
    B = to_device(B_np, w["layout"], device)
    alg = F.load_alg(w["alg"])
    lib_comm = F.Comm.from_torch_distributed(device=device.index) if (world > 1 and args.combine == "lib") else None
    plan = F.Plan(alg, P, Q, N, L, layout=w["layout"], strategy=args.strategy, cse=bool(args.cse),
                  shard_rank=rank, shard_count=world, fuse=bool(args.fuse), collapse=bool(args.collapse),
                  comm=lib_comm, root="slabs" if args.output == "slabs" else 0, shard_mode=args.shard_mode)
    # --combine p2p: the partial C lives in a peer-mapped buffer and one pull-reduce kernel per rank
    # sums its slab over every rank's partial (fmm_p2p_*, CUDA IPC over NVLink, no NCCL data path)
    p2p = out_slab = None
    outer, inner = (P, N) if w["layout"] == "row" else (N, P)
    if world > 1 and args.combine == "p2p":
        p2p = F.P2P.from_torch_distributed(8 * P * N, device=device.index)
        C = p2p.partial(P, N, w["layout"])
        s0, s1 = F.dist_slab(P, N, w["layout"], world, rank)
        out_slab = torch.empty(s1 - s0, inner, dtype=torch.float64, device=device)
    else:
        C = plan.new_output()
    st = plan.stats()
    dmma_peak, dfma_peak = F.probe_fp64_peak()
    stream = torch.cuda.current_stream()

    def combine():
        if lib_comm is not None:  # a distributed plan reduces inside fmm_execute
            return
        if p2p is not None:
            stream.synchronize()
            dist.barrier()  # every partial complete
            p2p.reduce_slab(outer, inner, out_slab, stream=stream)
            stream.synchronize()
            dist.barrier()  # every slab read before the next step overwrites a partial
        elif args.output == "slabs":
            scatter_partials(C)
        else:
            combine_partials(C)

    def step(evs=None):
        if evs is None:
            plan.execute(A, B, C, stream=stream)
        else:
            plan.execute_events(A, B, C, evs[:4], stream=stream)
        combine()
        if evs is not None:
            evs[4].record(stream)  # after the combine: the comm share of a step (N > 1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    for e in (x for row in evs for x in row):
        e.record(stream)  # torch creates the underlying cudaEvent_t lazily, at the first record
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(device.index)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    flops = 2.0 * P * Q * N
    value = flops / (ms_step * 1e-3) / 1e9

    # result check after the timed steps (C holds the last step's combined product): sampled rows
    # of rank 0's part of C against a cuBLAS product of the same rows (a check, not a timing), at the
    # north-star tolerance max |C - AB| <= 1e-10 ||A||_F ||B||_F
    check = None
    if rank == 0:
        if (args.output == "slabs" or p2p is not None) and world > 1:
            lo, hi = F.dist_slab(P, N, w["layout"], world, 0)
        else:
            lo, hi = 0, (P if w["layout"] == "row" else N)
        g = torch.Generator().manual_seed(7)
        idx = torch.randint(lo, max(lo + 1, hi), (min(64, max(hi - lo, 1)),), generator=g).to(device)
        if hi > lo:
            # rank 0's result: C itself, or (p2p) its reduced slab of C's storage rows
            got = (lambda rows: out_slab[rows - lo]) if p2p is not None else (
                (lambda rows: C[rows]) if w["layout"] == "row" else (lambda cols: C[:, cols].t()))
            if w["layout"] == "row":
                err = (got(idx) - A[idx] @ B).abs().max().item()
            else:  # slabs of C's columns
                err = (got(idx) - (A @ B[:, idx]).t()).abs().max().item()
            tol = 1e-10 * torch.linalg.norm(A).item() * torch.linalg.norm(B).item()
            check = {"sampled": int(idx.numel()), "of": "rows" if w["layout"] == "row" else "columns",
                     "max_abs_err": err, "tolerance": tol, "ok": bool(err <= tol)}

    # per-phase device times measured on the launching stream during the timed region
    ph = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]), e[3].elapsed_time(e[4])]
                   for e in evs])
    form_ms, gemm_ms, asm_ms, comm_ms = [float(x) for x in ph.mean(axis=0)]
    add_ms = form_ms + asm_ms
    peaks, peak_src = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", HBM_FALLBACK))
    fused = st.get("fused_launches", 0) > 0
    # leaf-product flops of the dominant launch (the fused leaf level, or the plain leaf GEMM)
    gemm_tf = st["leaf_flops"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    sep_bytes = st["add_bytes"] - st["fused_add_bytes"]
    add_gbs = sep_bytes / (add_ms * 1e-3) / 1e9 if add_ms > 0 else None

    # the other leaf-level schedule on the same workload: with --fuse 0 (default) the fused
    # leaf-level launch (level-L formation / leaf GEMM / level-L assembly in one cooperative
    # kernel, addition CTAs on their own SMs), with --fuse 1 the separate kernels
    other = None
    if not args.no_other and L >= 1:
        try:
            plan_o = F.Plan(alg, P, Q, N, L, layout=w["layout"], strategy=args.strategy, cse=bool(args.cse),
                            shard_rank=rank, shard_count=world, fuse=not fused, collapse=False)
            so = plan_o.stats()
            for _ in range(2):
                plan_o.execute(A, B, C, stream=stream)
            nu = max(3, min(args.steps, 10))
            evu = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(nu)]
            for e in (x for row in evu for x in row):
                e.record(stream)  # creates the underlying cudaEvent_t
            torch.cuda.synchronize()
            for k in range(nu):
                plan_o.execute_events(A, B, C, evu[k], stream=stream)
            torch.cuda.synchronize()
            phu = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3]),
                             e[0].elapsed_time(e[3])] for e in evu]).mean(axis=0)
            o_fused = so.get("fused_launches", 0) > 0
            other = {"fused_leaf_level": o_fused, "collapsed_levels": bool(so.get("collapsed", 0)), "ms_per_step": float(phu[3]), "value": flops / (phu[3] * 1e-3) / 1e9,
                     "steps": nu, "phases_ms": {"formation": float(phu[0]), "leaf_level": float(phu[1]),
                                                "assembly_and_strips": float(phu[2])},
                     "launches": so["launches"]}
            del plan_o
            plan.execute(A, B, C, stream=stream)  # C holds the headline path's result again
        except Exception as e:  # an optional extra measurement must not cost the bench line
            other = {"error": str(e)[:200]}
            torch.cuda.synchronize()

    # shape matching (fmm_select over every algorithm file x its six Prop. 1/2 permutations x L <= 3,
    # by the library's cost model) on the same inputs: what the paper's "match the shape" buys here
    shape_matched = None
    if not args.no_other and rank == 0 and world == 1:
        import glob
        cands = [F.load_alg(os.path.basename(x)[:-4]) for x in sorted(glob.glob(os.path.join(ROOT, "algs", "*.txt")))]
        sel, sel_L, sel_pred = F.select(cands, P, Q, N, 3, w["layout"])
        if sel is not None:
            try:
                plan_s = F.Plan(sel, P, Q, N, sel_L, layout=w["layout"], strategy=args.strategy, cse=bool(args.cse))
                for _ in range(2):
                    plan_s.execute(A, B, C, stream=stream)
                ns = max(3, min(args.steps, 10))
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                for _ in range(ns):
                    plan_s.execute(A, B, C, stream=stream)
                s1.record(stream)
                torch.cuda.synchronize()
                ms_s = s0.elapsed_time(s1) / ns
                shape_matched = {"algorithm": sel.name, "base_case": [sel.M, sel.K, sel.N], "rank": sel.R, "levels": sel_L,
                                 "predicted_ms": sel_pred, "ms_per_step": ms_s, "value": flops / (ms_s * 1e-3) / 1e9,
                                 "steps": ns, "note": "not the headline: BASELINE fixes the algorithm and L"}
                del plan_s
                plan.execute(A, B, C, stream=stream)
            except Exception as e:  # optional, like other_schedule
                shape_matched = {"algorithm": sel.name, "levels": sel_L, "error": str(e)[:200]}

    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(args.workload, {}).get("grouped_dgemm_bytes_per_launch")
    except OSError:
        pass
    kname = ("grouped_dgemm_tma<FUSED> (level-L formation + leaf products on DMMA mma.sync.m8n8k4.f64 + "
             "level-L assembly, one persistent launch)" if fused else
             "grouped_dgemm_tma (leaf products, mma.sync.m8n8k4.f64 = DMMA)")
    roofline = {"bound": "tensor", "kernel": kname,
                "achieved": gemm_tf, "peak": dmma_peak, "unit": "TFLOP/s",
                "frac": (gemm_tf / dmma_peak) if gemm_tf else None, "traffic": traffic,
                "peak_source": "in-run DMMA microbenchmark fmm_probe_fp64_peak (MEASURED_PEAKS.json has no FP64 "
                               "figure; nameplate 148 SM x 128 flop/clk x 1.965 GHz = 37.2)",
                "algorithmic_flops_per_launch": st["leaf_flops"],
                "hidden_addition_bytes_per_launch": st["fused_add_bytes"]}

    # cuBLAS DGEMM (classical) on the same inputs, same box: the comparison point
    cub = None
    if rank == 0:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ref = torch.matmul(A, B)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0.record(); torch.matmul(A, B); e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        cub = flops / (best * 1e-3) / 1e9
        del ref

    # the classical comparison on our own DMMA GEMM (L = 0): at N > 1 each rank multiplies its row
    # slab of A by B with no exchange (SURVEY f1's classical row-slab split), timed as max over ranks
    own = None
    try:
        if w["layout"] == "row":
            r0, r1 = F.dist_slab(P, N, "row", world, rank)
            As = A[r0:r1]
        else:  # column-major: the slab of C's columns, i.e. B's columns
            r0, r1 = F.dist_slab(P, N, "col", world, rank)
            As = None
        m_rows = (r1 - r0) if As is not None else P
        n_cols = N if As is not None else (r1 - r0)
        cp = F.Plan(alg, m_rows, Q, n_cols, 0, layout=w["layout"])
        Aa, Bb = (As, B) if As is not None else (A, B[:, r0:r1])
        Cc = cp.new_output()
        for _ in range(2):
            cp.execute(Aa, Bb, Cc, stream=stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            cp.execute(Aa, Bb, Cc, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        tt = torch.tensor([e0.elapsed_time(e1) / 3], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        own = {"ms": float(tt.item()), "value": flops / (float(tt.item()) * 1e-3) / 1e9,
               "what": "classical DMMA GEMM (L = 0, this library)" + (f", row slabs x{world}, no exchange" if world > 1 else "")}
        del cp, Cc
    except Exception as ex:  # noqa: BLE001  (a comparison leg only)
        own = {"error": str(ex)[:200]}

    # end-to-end through the public host-buffer API: H2D of A and B, execute, D2H of C per step
    e2e = None
    if not args.no_e2e:
        def pinned(x, rows, cols):
            if w["layout"] == "row":
                return (torch.from_numpy(np.ascontiguousarray(x)) if x is not None
                        else torch.empty(rows, cols, dtype=torch.float64)).pin_memory()
            return (torch.from_numpy(np.ascontiguousarray(x.T)) if x is not None
                    else torch.empty(cols, rows, dtype=torch.float64)).pin_memory().t()
        Ah, Bh, Ch = pinned(A_np, P, Q), pinned(B_np, Q, N), pinned(None, P, N)
        h2d = 8 * (P * Q + Q * N)
        d2h = 8 * P * N if rank == 0 else 0
        slab_h = None
        if p2p is not None and rank == 0:  # rank 0's result is its reduced slab
            slab_h = torch.empty(tuple(out_slab.shape), dtype=torch.float64, pin_memory=True)
            d2h = 8 * out_slab.numel()
        def e2e_step():
            if world == 1:
                # pipelined public host API: H2D of this step, compute, D2H of its C
                plan.execute_host(Ah, Bh, Ch, stream=stream, asynchronous=True)
            else:
                A.copy_(Ah, non_blocking=True); B.copy_(Bh, non_blocking=True)
                plan.execute(A, B, C, stream=stream)
                combine()
                if rank == 0:
                    if slab_h is not None:
                        slab_h.copy_(out_slab, non_blocking=True)
                    else:
                        Ch.copy_(C, non_blocking=True)
                torch.cuda.synchronize()
        e2e_step()
        plan.sync()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        n_e2e = max(3, min(max(args.steps, 30), 60))  # fill and drain of the copy pipeline amortised over >= 30 steps
        h0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        plan.sync()
        torch.cuda.synchronize()
        ms_e = (time.perf_counter() - h0) * 1e3
        if world > 1:
            tt = torch.tensor([ms_e], dtype=torch.float64, device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms_e = float(tt.item())
        e2e = {"value": flops / (ms_e / n_e2e * 1e-3) / 1e9, "unit": "GFLOPS", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ms_e / n_e2e, "steps": n_e2e,
               "timing": "host wall clock over the steps, device synchronised on both sides",
               "api": "fmm_execute_host_async x steps + fmm_sync (pinned host A, B, C; copy-in, compute and "
                      "copy-out of consecutive steps overlap)" if world == 1 else
               "H2D + fmm_execute + NCCL reduce + D2H"}

    # N > 1: the replication of A and B from rank 0, timed on its own after the timed
    # region (every rank holds the seeded inputs, so the steps above do not include it)
    bcast = None
    if world > 1:
        from paper_1409_2908_b200.dist import storage_view
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        dist.barrier()
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(reps):
            dist.broadcast(storage_view(A), src=0)
            dist.broadcast(storage_view(B), src=0)
        b1.record(stream)
        torch.cuda.synchronize()
        tb = torch.tensor([b0.elapsed_time(b1) / reps], dtype=torch.float64, device=device)
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        bms = float(tb.item())
        bbytes = 8.0 * (P * Q + Q * N)
        bcast = {"ms": bms, "bytes": bbytes, "algbw_gbs": bbytes / (bms * 1e-3) / 1e9,
                 "value_with_broadcast": flops / ((ms_step + bms) * 1e-3) / 1e9}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O
        O.build()
        cpu = cpu_oracle_sample(w, A_np, B_np, args.cpu_frac)
        cpu.pop("seconds", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": w["desc"], "algorithm": w["alg"], "rank": alg.R, "levels": L, "P": P, "Q": Q,
                       "N": N, "layout": w["layout"], "inputs": "uniform[-1,1) fp64, numpy PCG64 seeds 0 (A), 1 (B)",
                       "strategy": args.strategy, "cse": bool(args.cse),
                       "l2": "inputs larger than L2 (A, B, C 0.54 GB each vs 126 MB); no flush"
                       if args.workload != "c1" else "small config: L2-resident",
                       "parallelism": ((f"{args.shard_mode}-level shards x{world} + peer-memory slab reduce "
                                        "(fmm_p2p: one pull kernel per rank over CUDA IPC)") if p2p is not None else
                                       (f"{args.shard_mode}-level shards x{world} + {args.dist_backend.upper()} "
                                        f"{'reduce to rank 0' if args.output == 'root' else 'slab reduce-scatter'} "
                                        f"({'fmm_execute' if lib_comm else 'torch.distributed'})")
                                       if world > 1 else "1 GPU"),
                       "fused_leaf_level": fused, "collapsed_levels": bool(st.get("collapsed", 0)),
                       **({"dist_backend": "gloo (control-flow check, ranks share a GPU: NOT a measurement)"}
                          if world > 1 and args.dist_backend == "gloo" else {})},
            "roofline": roofline,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": int(st["launches"]) * args.steps,
            "cpu_baseline": cpu,
            "phases_ms": {"formation_levels_below_L" if fused else "formation": form_ms,
                          "fused_leaf_level" if fused else "leaf_gemm": gemm_ms,
                          "assembly_and_strips": add_ms - form_ms,
                          "combine_reduce": comm_ms if world > 1 else 0.0},
            "input_broadcast": bcast,
            "combine_algbw_gbs": (8.0 * P * N / (comm_ms * 1e-3) / 1e9) if world > 1 and comm_ms else None,
            "additions": {"algorithmic_bytes_per_step": st["add_bytes"],
                          "bytes_in_fused_launch": st["fused_add_bytes"],
                          "separate_kernel_bytes": sep_bytes, "separate_kernel_gbs": add_gbs, "peak_gbs": hbm,
                          "separate_kernel_frac": (add_gbs / hbm) if add_gbs else None, "peak_source": peak_src},
            "other_schedule": other,
            "shape_matched": shape_matched,
            "fp64_peak_tflops": {"dmma_measured": dmma_peak, "dfma_measured": dfma_peak, "nameplate": 37.2},
            "effective_frac_of_fp64_peak": value / 1e3 / dmma_peak,
            "cublas_dgemm_gflops_same_inputs": cub,
            "classical_own_dgemm": own,
            "result_check": check,
            "paper_effective_gflops": (2.0 * P * Q * N - P * N) / (ms_step * 1e-3) / 1e9,
            "plan": {k: st[k] for k in ("gemm_flops", "add_flops", "add_bytes", "launches", "leaves")},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
