#!/usr/bin/env python
"""bench.py — effective FP64 GFLOPS (2MKN/t) of the recursive fast matrix multiplication hot path
(arXiv 1409.2908) on B200, through the repo's C-ABI library.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

One step = one fmm_execute of the whole hot path (S/T formation at every level, the grouped DMMA
leaf GEMM, C assembly at every level, peel strips) over one synthetic input pair already
resident in HBM; for N > 1 each rank computes its leaf shard and the partial C are summed inside
the same fmm_execute (the library's distributed plan: NCCL reduce in overlapped row chunks, or
the peer-memory combine), inside the timed region.  Prints ONE JSON line on rank 0.

--gpus N > 1 without torchrun (WORLD_SIZE unset) re-launches this script under
torch.distributed.run with N ranks; under torchrun, --gpus must equal WORLD_SIZE.

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
    ap.add_argument("--shard-mode", default="leaf", choices=["leaf", "top", "slab"],
                    help="N > 1: leaf-level HYBRID sharding or the top-level products in contiguous ranges (partial "
                         "C per rank, combined); or slab: each rank runs the whole method on its slab of C's rows "
                         "(columns when column-major), nothing to combine")
    ap.add_argument("--combine", default="auto", choices=["auto", "lib", "p2p", "p2p_push", "torch"],
                    help="N > 1: the partial-C combine.  lib: NCCL inside fmm_execute (fmm_plan_create_dist, "
                         "row chunks overlapped with the assembly); p2p: the peer-memory pull-reduce inside "
                         "fmm_execute (fmm_plan_create_p2p); p2p_push: the kernels that write C store each "
                         "rank's partial into the root's buffer over peer memory, the root sums (root output); "
                         "torch: torch.distributed.reduce after fmm_execute.  "
                         "auto = lib with --dist-backend nccl, p2p with gloo")
    ap.add_argument("--output", default="root", choices=["root", "slabs"],
                    help="N > 1: C summed onto rank 0, or slab-distributed (slab g of C summed onto rank g)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1: gloo only to exercise the multi-rank control flow where ranks share a GPU (not a measurement)")
    ap.add_argument("--no-other", action="store_true", help="skip timing the other leaf-level schedule (fused vs separate)")
    ap.add_argument("--configs", default="auto",
                    help="extra BASELINE configs timed after the headline, one sub-record each (comma list, "
                         "'none'); auto = c3,c4,c5t,c5 for the default c2 run at N = 1")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.combine == "auto":
        args.combine = "p2p" if args.dist_backend == "gloo" else "lib"
    w = WORKLOADS[args.workload]
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None and int(world_env) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}: launch one rank per GPU\n")
        sys.exit(2)
    if world_env is None and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    if args.impl == "reference":
        run_reference(args, w)
        return
    Run(args, w).go()


def relaunch(n: int) -> int:
    """Run this script again under torch.distributed.run with n ranks (one per GPU, 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


class Run:
    """One bench invocation of our arm: set-up, the timed steps, the comparison legs, the JSON line.
    State shared by the legs lives on the instance."""

    def __init__(self, args, w):
        import torch
        import torch.distributed as dist
        self.args, self.w = args, w
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world > 1:
            # NCCL's init lines (communicator ranks, NVLS) in the log: the driver counts ranks from them
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
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
        self.device = torch.device(f"cuda:{torch.cuda.current_device()}")
        import __graft_entry__
        __graft_entry__.build()
        import paper_1409_2908_b200 as F
        self.F = F
        self.P, self.Q, self.N, self.L = w["P"], w["Q"], w["N"], w["L"]
        self.flops = 2.0 * self.P * self.Q * self.N

    # ---- set-up ------------------------------------------------------------------------------
    def setup(self):
        args, w, F, torch = self.args, self.w, self.F, self.torch
        P, Q, N, L, world, rank, device = self.P, self.Q, self.N, self.L, self.world, self.rank, self.device
        self.A_np, self.B_np = gen_inputs(w)
        self.slab = world > 1 and args.shard_mode == "slab"
        self.Pp, self.Np = P, N  # this rank's plan dimensions (slab mode: its slab of C)
        self.Ax_np, self.Bx_np = self.A_np, self.B_np
        if self.slab:
            r0, r1 = F.dist_slab(P, N, w["layout"], world, rank)
            self.slab_range = (r0, r1)
            if w["layout"] == "row":
                self.Ax_np, self.Pp = self.A_np[r0:r1], r1 - r0
            else:
                self.Bx_np, self.Np = self.B_np[:, r0:r1], r1 - r0
        self.A = to_device(self.Ax_np, w["layout"], device)
        self.B = to_device(self.Bx_np, w["layout"], device)
        self.alg = F.load_alg(w["alg"])
        # N > 1: the combine runs inside fmm_execute -- NCCL (lib, fmm_plan_create_dist) or the
        # peer-memory pull-reduce over CUDA IPC (p2p, fmm_plan_create_p2p) -- or after it (torch)
        combined = world > 1 and not self.slab
        self.lib_comm = F.Comm.from_torch_distributed(device=device.index) if (combined and args.combine == "lib") else None
        push = args.combine == "p2p_push" and args.output != "slabs"
        p2p_bytes = 8 * ((P * N + 1) // 2 * 2) * (world if push else 1)  # push: G partial slots on the root
        self.p2p = (F.P2P.from_torch_distributed(p2p_bytes, device=device.index)
                    if (combined and args.combine in ("p2p", "p2p_push")) else None)
        if self.slab:  # the whole method on this rank's slab: an ordinary single-GPU plan
            self.plan = F.Plan(self.alg, self.Pp, Q, self.Np, L, layout=w["layout"], strategy=args.strategy,
                               cse=bool(args.cse), fuse=bool(args.fuse), collapse=bool(args.collapse))
        else:
            self.plan = F.Plan(self.alg, P, Q, N, L, layout=w["layout"], strategy=args.strategy, cse=bool(args.cse),
                               shard_rank=rank, shard_count=world, fuse=bool(args.fuse), collapse=bool(args.collapse),
                               comm=self.lib_comm, p2p=self.p2p, barrier=(self.dist.barrier if self.p2p else None),
                               root="slabs" if args.output == "slabs" else 0, shard_mode=args.shard_mode,
                               p2p_push=push if self.p2p else None)
        self.outer, self.inner = (P, N) if w["layout"] == "row" else (N, P)
        self.C = self.plan.new_output()
        self.st = self.plan.stats()
        self.fused = self.st.get("fused_launches", 0) > 0
        self.dmma_peak, self.dfma_peak = F.probe_fp64_peak()
        self.stream = torch.cuda.current_stream()

    def combine(self):
        from paper_1409_2908_b200.dist import combine_partials, scatter_partials
        if self.world == 1 or self.slab or self.args.combine != "torch":  # lib / p2p combine inside fmm_execute
            return
        if self.args.output == "slabs":
            scatter_partials(self.C)
        else:
            combine_partials(self.C)

    def step(self):
        self.plan.execute(self.A, self.B, self.C, stream=self.stream)
        self.combine()

    def max_over_ranks(self, ms):
        if self.world > 1:
            tt = self.torch.tensor([ms], dtype=self.torch.float64, device=self.device)
            self.dist.all_reduce(tt, op=self.dist.ReduceOp.MAX)
            ms = float(tt.item())
        return ms

    # ---- the timed region ----------------------------------------------------------------------
    def timed_steps(self):
        # the headline: whole-step events around K plain fmm_execute calls (the library's default
        # path, CUDA-graph replay where the plan allows it), max over ranks
        torch, args, stream = self.torch, self.args, self.stream
        for _ in range(args.warmup):
            self.step()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(self.device.index)
        clocks.start()
        time.sleep(0.3)
        if self.world > 1:
            self.dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        for k in range(args.steps):
            self.step()
        t1.record(stream)
        torch.cuda.synchronize()
        if self.world > 1:
            self.dist.barrier()
        self.clk = clocks.stop()
        self.ms_step = self.max_over_ranks(t0.elapsed_time(t1)) / args.steps
        self.value = self.flops / (self.ms_step * 1e-3) / 1e9

    def phase_split(self, reps=5):
        # per-phase device times from a separate pass (fmm_execute_timed: plain launches with an
        # event after each; formation / leaf products / assembly / peel strips / exposed combine),
        # median of `reps` passes after an untimed one
        import numpy as np
        ph = []
        for it in range(reps + 1):
            if self.world > 1 and self.args.combine == "torch":
                _, t = self.plan.execute_timed(self.A, self.B, self.C, stream=self.stream)
                e0 = self.torch.cuda.Event(enable_timing=True)
                e1 = self.torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                self.combine()
                e1.record(self.stream)
                e1.synchronize()
                t["total_ms"] += e0.elapsed_time(e1)
            else:
                _, t = self.plan.execute_timed(self.A, self.B, self.C, stream=self.stream)
            if it:
                ph.append([t["formation_ms"], t["gemm_ms"], t["assembly_ms"], t["strips_ms"], t["total_ms"]])
        m = np.median(np.array(ph), axis=0)
        self.form_ms, self.gemm_ms, self.asm_ms, self.strip_ms, tot = [float(x) for x in m]
        self.comm_ms = max(0.0, tot - self.form_ms - self.gemm_ms - self.asm_ms - self.strip_ms) if self.world > 1 else 0.0

    def result_check(self):
        # after the timed steps C holds the last step's combined product: sampled rows of rank 0's
        # part of C against a cuBLAS product of the same rows (a check, not a timing), at the
        # north-star tolerance max |C - AB| <= 1e-10 ||A||_F ||B||_F
        if self.rank != 0:
            return None
        torch, w, F, A, B, C = self.torch, self.w, self.F, self.A, self.B, self.C
        if self.slab:  # rank 0's own slab, against its slab of A (rows) or B (columns)
            lo, hi = 0, (self.Pp if w["layout"] == "row" else self.Np)
        elif self.args.output == "slabs" and self.world > 1:
            lo, hi = F.dist_slab(self.P, self.N, w["layout"], self.world, 0)
        else:
            lo, hi = 0, (self.P if w["layout"] == "row" else self.N)
        if hi <= lo:
            return None
        g = torch.Generator().manual_seed(7)
        idx = torch.randint(lo, max(lo + 1, hi), (min(64, max(hi - lo, 1)),), generator=g).to(self.device)
        if w["layout"] == "row":
            got = lambda rows: C[rows]  # noqa: E731
        else:
            got = lambda cols: C[:, cols].t()  # noqa: E731
        if w["layout"] == "row":
            err = (got(idx) - A[idx] @ B).abs().max().item()
        else:  # slabs of C's columns
            err = (got(idx) - (A @ B[:, idx]).t()).abs().max().item()
        tol = 1e-10 * torch.linalg.norm(A).item() * torch.linalg.norm(B).item()
        return {"sampled": int(idx.numel()), "of": "rows" if w["layout"] == "row" else "columns",
                "max_abs_err": err, "tolerance": tol, "ok": bool(err <= tol)}

    # ---- comparison legs (outside the timed region) --------------------------------------------
    def other_schedule(self):
        # the other leaf-level schedule on the same workload: with --fuse 0 (default) the fused
        # leaf-level launch (level-L formation / leaf GEMM / level-L assembly in one cooperative
        # kernel, addition CTAs on their own SMs), with --fuse 1 the separate kernels
        import numpy as np
        args, torch, stream = self.args, self.torch, self.stream
        if args.no_other or self.L < 1 or self.slab:
            return None
        try:
            plan_o = self.F.Plan(self.alg, self.P, self.Q, self.N, self.L, layout=self.w["layout"],
                                 strategy=args.strategy, cse=bool(args.cse), shard_rank=self.rank,
                                 shard_count=self.world, fuse=not self.fused, collapse=False)
            so = plan_o.stats()
            for _ in range(2):
                plan_o.execute(self.A, self.B, self.C, stream=stream)
            nu = max(3, min(args.steps, 10))
            rows = []
            for k in range(nu):
                _, t = plan_o.execute_timed(self.A, self.B, self.C, stream=stream)
                rows.append([t["formation_ms"], t["gemm_ms"], t["assembly_ms"] + t["strips_ms"], t["total_ms"]])
            phu = np.array(rows).mean(axis=0)
            other = {"fused_leaf_level": so.get("fused_launches", 0) > 0, "collapsed_levels": bool(so.get("collapsed", 0)),
                     "ms_per_step": float(phu[3]), "value": self.flops / (phu[3] * 1e-3) / 1e9,
                     "steps": nu, "phases_ms": {"formation": float(phu[0]), "leaf_level": float(phu[1]),
                                                "assembly_and_strips": float(phu[2])},
                     "launches": so["launches"]}
            del plan_o
            self.plan.execute(self.A, self.B, self.C, stream=stream)  # C holds the headline path's result again
            return other
        except Exception as e:  # an optional extra measurement must not cost the bench line
            torch.cuda.synchronize()
            return {"error": str(e)[:200]}

    def shape_matched(self):
        # shape matching (fmm_select over every algorithm file x its six Prop. 1/2 permutations x
        # L <= 3, by the library's cost model) on the same inputs: what the paper's "match the shape"
        # buys here
        import glob
        args, torch, stream, F = self.args, self.torch, self.stream, self.F
        if args.no_other or self.rank != 0 or self.world != 1:
            return None
        cands = [F.load_alg(os.path.basename(x)[:-4]) for x in sorted(glob.glob(os.path.join(ROOT, "algs", "*.txt")))]
        sel, sel_L, sel_pred = F.select(cands, self.P, self.Q, self.N, 3, self.w["layout"])
        if sel is None:
            return None
        try:
            plan_s = F.Plan(sel, self.P, self.Q, self.N, sel_L, layout=self.w["layout"], strategy=args.strategy,
                            cse=bool(args.cse))
            for _ in range(2):
                plan_s.execute(self.A, self.B, self.C, stream=stream)
            ns = max(3, min(args.steps, 10))
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(ns):
                plan_s.execute(self.A, self.B, self.C, stream=stream)
            s1.record(stream)
            torch.cuda.synchronize()
            ms_s = s0.elapsed_time(s1) / ns
            del plan_s
            self.plan.execute(self.A, self.B, self.C, stream=stream)
            return {"algorithm": sel.name, "base_case": [sel.M, sel.K, sel.N], "rank": sel.R, "levels": sel_L,
                    "predicted_ms": sel_pred, "ms_per_step": ms_s, "value": self.flops / (ms_s * 1e-3) / 1e9,
                    "steps": ns, "note": "not the headline: BASELINE fixes the algorithm and L"}
        except Exception as e:  # optional, like other_schedule
            return {"algorithm": sel.name, "levels": sel_L, "error": str(e)[:200]}

    def cublas(self):
        # cuBLAS DGEMM (classical) on the same inputs, same box: the comparison point
        if self.rank != 0:
            return None
        torch, A, B = self.torch, self.A, self.B
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.matmul(A, B)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0.record()
            torch.matmul(A, B)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return self.flops / (best * 1e-3) / 1e9

    def shard_scaling(self):
        # N = 1 only: the compute side of the multi-GPU split, measured on this GPU -- for G = 2, 4, 8
        # every shard plan of the headline workload (leaf-level HYBRID shards, then top-level product
        # ranges) runs here in turn; max_g t_g against t_1 / G is the load balance a G-GPU run would
        # see before its combine.  The combine itself (NCCL / peer memory over NVLink) is not
        # measurable on one GPU: its volume is the partial C per rank, reported beside.
        args, torch, stream, F = self.args, self.torch, self.stream, self.F
        if self.world != 1 or args.no_other:
            return None
        out = {"what": "per-shard device time of the headline workload's shard plans, run one after another on "
                       "this GPU (compute only; no combine)", "t1_ms": self.ms_step, "G": {}}
        try:
            for mode in ("leaf", "top"):
                for G in (2, 4, 8):
                    ts = []
                    for g in range(G):
                        p = F.Plan(self.alg, self.P, self.Q, self.N, self.L, layout=self.w["layout"], shard_rank=g,
                                   shard_count=G, shard_mode=mode)
                        for _ in range(3):
                            p.execute(self.A, self.B, self.C, stream=stream)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        torch.cuda.synchronize()
                        e0.record(stream)
                        for _ in range(5):
                            p.execute(self.A, self.B, self.C, stream=stream)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1) / 5)
                        del p
                    tmax = max(ts)
                    out["G"][f"{mode}{G}"] = {"shard_ms": ts, "max_ms": tmax, "mean_ms": sum(ts) / G,
                                             "balance_max_over_mean": tmax / (sum(ts) / G),
                                             "compute_efficiency": self.ms_step / (G * tmax),
                                             "partial_C_bytes_per_rank": 8.0 * self.P * self.N}
            # the other partition, for comparison: each rank runs the whole method on its slab of C
            # (rows of a row-major C, columns of a column-major one: A's rows or B's columns), so no
            # partial products exist and nothing is combined; every rank reads all of B (all of A)
            lay = self.w["layout"]
            for G in (2, 4, 8):
                ts = []
                for g in range(G):
                    r0, r1 = F.dist_slab(self.P, self.N, lay, G, g)
                    if lay == "row":
                        p = F.Plan(self.alg, r1 - r0, self.Q, self.N, self.L, layout=lay)
                        a_, b_, c_ = self.A[r0:r1], self.B, self.C[r0:r1]
                    else:
                        p = F.Plan(self.alg, self.P, self.Q, r1 - r0, self.L, layout=lay)
                        a_, b_, c_ = self.A, self.B[:, r0:r1], self.C[:, r0:r1]
                    for _ in range(3):
                        p.execute(a_, b_, c_, stream=stream)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record(stream)
                    for _ in range(5):
                        p.execute(a_, b_, c_, stream=stream)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 5)
                    del p
                tmax = max(ts)
                out["G"][f"slab{G}"] = {"shard_ms": ts, "max_ms": tmax, "mean_ms": sum(ts) / G,
                                       "balance_max_over_mean": tmax / (sum(ts) / G),
                                       "compute_efficiency": self.ms_step / (G * tmax), "partial_C_bytes_per_rank": 0.0}
            self.plan.execute(self.A, self.B, self.C, stream=stream)  # C holds the headline result again
            torch.cuda.synchronize()
        except Exception as ex:  # noqa: BLE001  (a comparison leg only)
            out["error"] = str(ex)[:200]
        return out

    def own_classical(self):
        # the classical comparison on our own DMMA GEMM (L = 0): at N > 1 each rank multiplies its
        # row slab of A by B with no exchange (SURVEY f1's classical row-slab split), max over ranks
        torch, F, w, A, B, stream = self.torch, self.F, self.w, self.A, self.B, self.stream
        if self.slab:
            return None  # slab mode already is the row / column-slab split (with the fast method)
        try:
            lay = w["layout"]
            r0, r1 = F.dist_slab(self.P, self.N, lay, self.world, self.rank)
            if lay == "row":
                cp = F.Plan(self.alg, r1 - r0, self.Q, self.N, 0, layout=lay)
                Aa, Bb = A[r0:r1], B
            else:  # column-major: the slab of C's columns, i.e. B's columns
                cp = F.Plan(self.alg, self.P, self.Q, r1 - r0, 0, layout=lay)
                Aa, Bb = A, B[:, r0:r1]
            Cc = cp.new_output()
            for _ in range(2):
                cp.execute(Aa, Bb, Cc, stream=stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if self.world > 1:
                self.dist.barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(3):
                cp.execute(Aa, Bb, Cc, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = self.max_over_ranks(e0.elapsed_time(e1) / 3)
            del cp, Cc
            return {"ms": ms, "value": self.flops / (ms * 1e-3) / 1e9,
                    "what": "classical DMMA GEMM (L = 0, this library)" +
                            (f", row slabs x{self.world}, no exchange" if self.world > 1 else "")}
        except Exception as ex:  # noqa: BLE001  (a comparison leg only)
            return {"error": str(ex)[:200]}

    def e2e(self):
        # end to end through the public host-buffer API: H2D of A and B, execute, D2H of C per step
        import numpy as np
        args, torch, w, world, rank = self.args, self.torch, self.w, self.world, self.rank
        if args.no_e2e:
            return None
        P, Q, N = self.Pp, self.Q, self.Np  # this rank's problem (all of it unless slab mode)

        def pinned(x, rows, cols):
            if w["layout"] == "row":
                return (torch.from_numpy(np.ascontiguousarray(x)) if x is not None
                        else torch.empty(rows, cols, dtype=torch.float64)).pin_memory()
            return (torch.from_numpy(np.ascontiguousarray(x.T)) if x is not None
                    else torch.empty(cols, rows, dtype=torch.float64)).pin_memory().t()
        Ah, Bh, Ch = pinned(self.Ax_np, P, Q), pinned(self.Bx_np, Q, N), pinned(None, P, N)
        h2d = 8 * (P * Q + Q * N)
        d2h = 8 * P * N if (rank == 0 or self.slab) else 0

        def e2e_step():
            if world == 1:
                # pipelined public host API: H2D of this step, compute, D2H of its C
                self.plan.execute_host(Ah, Bh, Ch, stream=self.stream, asynchronous=True)
            else:
                self.A.copy_(Ah, non_blocking=True)
                self.B.copy_(Bh, non_blocking=True)
                self.plan.execute(self.A, self.B, self.C, stream=self.stream)
                self.combine()
                if rank == 0 or self.slab:  # slab mode: every rank downloads its slab of C
                    Ch.copy_(self.C, non_blocking=True)
                torch.cuda.synchronize()
        e2e_step()
        self.plan.sync()
        if world > 1:
            self.dist.barrier()
        torch.cuda.synchronize()
        n_e2e = 60  # the copy pipeline's fill (first upload) and drain (last download) amortised over 60 steps
        h0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        self.plan.sync()
        torch.cuda.synchronize()
        ms_e = self.max_over_ranks((time.perf_counter() - h0) * 1e3)
        combine_name = ("no combine: every rank multiplies its slab" if self.slab else
                        {"p2p": "peer-memory combine inside fmm_execute", "lib": "NCCL reduce inside fmm_execute",
                         "p2p_push": "peer-memory combine inside fmm_execute (partials pushed by the kernels)",
                         "torch": "torch.distributed reduce"}[self.args.combine])
        return {"value": self.flops / (ms_e / n_e2e * 1e-3) / 1e9, "unit": "GFLOPS", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e / n_e2e, "steps": n_e2e,
                "timing": "host wall clock over the steps, device synchronised on both sides",
                "api": "fmm_execute_host_async x steps + fmm_sync (pinned host A, B, C; copy-in, compute and "
                       "copy-out of consecutive steps overlap)" if world == 1 else
                f"H2D + fmm_execute ({combine_name}) + D2H"}

    def broadcast(self):
        # N > 1: the replication of the inputs from rank 0, timed on its own after the
        # timed region (every rank holds the seeded inputs, so the steps above do not include it).
        # With NCCL each rank receives only the top-level A / B blocks its plan reads
        # (fmm_plan_input_blocks: the blocks its level-1 products touch; everything for the owner of
        # the top-level peel strips), packed by rank 0 and sent point to point; with gloo (ranks
        # sharing a GPU) the whole of A and B is broadcast.
        if self.world == 1:
            return None
        import numpy as np
        from paper_1409_2908_b200.dist import storage_view
        torch, dist, stream = self.torch, self.dist, self.stream
        if self.slab:
            return self.broadcast_slabs()
        needA, needB, core, need_all = self.plan.input_blocks()
        needs = [None] * self.world
        dist.all_gather_object(needs, (needA, needB, need_all))
        a = self.alg
        P1, Q1, N1 = core
        pb, qb, nb = P1 // a.M, Q1 // a.K, N1 // a.N
        blocksA = [(i // a.K * pb, i % a.K * qb, pb, qb) for i in range(a.M * a.K)]
        blocksB = [(j // a.N * qb, j % a.N * nb, qb, nb) for j in range(a.K * a.N)]
        restricted = self.args.dist_backend == "nccl" and self.args.combine != "torch"
        reps = 3
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sent = 0.0
        if restricted:
            # (matrix, block) -> receivers; a receiver that reads everything gets whole matrices
            plan_ops = []
            for g in range(1, self.world):
                nA, nB, allg = needs[g]
                if allg:
                    plan_ops.append((g, "A", None))
                    plan_ops.append((g, "B", None))
                    continue
                plan_ops += [(g, "A", blocksA[i]) for i, f in enumerate(nA) if f]
                plan_ops += [(g, "B", blocksB[j]) for j, f in enumerate(nB) if f]
            mats = {"A": self.A, "B": self.B}

            def view(name, blk):
                X = mats[name]
                if blk is None:
                    return storage_view(X)
                r0, c0, rr, cc = blk
                return X[r0:r0 + rr, c0:c0 + cc]
            bufs = {}
            for op in plan_ops:
                if self.rank == 0 or self.rank == op[0]:
                    v = view(op[1], op[2])
                    bufs[op] = torch.empty(v.numel(), dtype=torch.float64, device=self.device)
            dist.barrier()
            torch.cuda.synchronize()
            b0.record(stream)
            for _ in range(reps):
                ops = []
                for op in plan_ops:
                    if self.rank == 0:
                        bufs[op].copy_(view(op[1], op[2]).reshape(-1))  # pack (strided block -> contiguous)
                        ops.append(dist.P2POp(dist.isend, bufs[op], op[0]))
                    elif self.rank == op[0]:
                        ops.append(dist.P2POp(dist.irecv, bufs[op], 0))
                if ops:
                    for w in dist.batch_isend_irecv(ops):
                        w.wait()
                for op in plan_ops:
                    if self.rank == op[0]:
                        v = view(op[1], op[2])
                        v.copy_(bufs[op].view(v.shape))  # unpack
            b1.record(stream)
            torch.cuda.synchronize()
            for op in plan_ops:
                sent += 8.0 * view(op[1], op[2]).numel()
            if self.rank == 0:
                del bufs
        else:
            dist.barrier()
            torch.cuda.synchronize()
            b0.record(stream)
            for _ in range(reps):
                dist.broadcast(storage_view(self.A), src=0)
                dist.broadcast(storage_view(self.B), src=0)
            b1.record(stream)
            torch.cuda.synchronize()
            sent = 8.0 * (self.P * self.Q + self.Q * self.N) * (self.world - 1)
        bms = self.max_over_ranks(b0.elapsed_time(b1) / reps)
        full = 8.0 * (self.P * self.Q + self.Q * self.N)
        return {"ms": bms, "bytes_sent": sent, "bytes_if_every_rank_got_everything": full * (self.world - 1),
                "restricted_to_blocks_read": restricted,
                "blocks_read_per_rank": [[int(sum(n[0])), int(sum(n[1])), bool(n[2])] for n in needs],
                "algbw_gbs": sent / (bms * 1e-3) / 1e9 if bms > 0 else None,
                "value_with_broadcast": self.flops / ((self.ms_step + bms) * 1e-3) / 1e9}

    def broadcast_slabs(self):
        # slab mode: the operand every rank needs whole (B for a row-major problem, A for a column-
        # major one) is broadcast; the other is cut into the ranks' slabs and sent point to point
        # (NCCL; with gloo the slabs are not sent)
        from paper_1409_2908_b200.dist import storage_view
        torch, dist, stream, w = self.torch, self.dist, self.stream, self.w
        row = w["layout"] == "row"
        whole = self.B if row else self.A
        full = to_device(self.A_np if row else self.B_np, w["layout"], self.device) if self.rank == 0 else None
        send = self.args.dist_backend == "nccl"
        own = self.A if row else self.B
        spans = [self.F.dist_slab(self.P, self.N, w["layout"], self.world, g) for g in range(self.world)]
        reps = 3
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(reps):
            dist.broadcast(storage_view(whole), src=0)
            if send:
                ops = []
                for g in range(1, self.world):
                    r0, r1 = spans[g]
                    if self.rank == 0:
                        part = full[r0:r1] if row else full[:, r0:r1]
                        ops.append(dist.P2POp(dist.isend, storage_view(part), g))
                    elif self.rank == g:
                        ops.append(dist.P2POp(dist.irecv, storage_view(own), 0))
                if ops:
                    for wk in dist.batch_isend_irecv(ops):
                        wk.wait()
        b1.record(stream)
        torch.cuda.synchronize()
        bms = self.max_over_ranks(b0.elapsed_time(b1) / reps)
        sent = 8.0 * whole.numel() * (self.world - 1) + (
            8.0 * sum((r1 - r0) for r0, r1 in spans[1:]) * (self.Q) if send else 0.0)
        return {"ms": bms, "bytes_sent": sent,
                "what": "broadcast of the operand every rank reads whole" + (" + its slab of the other, point to point"
                                                                             if send else " (gloo: slabs not sent)"),
                "algbw_gbs": sent / (bms * 1e-3) / 1e9 if bms > 0 else None,
                "value_with_broadcast": self.flops / ((self.ms_step + bms) * 1e-3) / 1e9}

    def roofline(self):
        st = self.st
        gemm_tf = st["leaf_flops"] / (self.gemm_ms * 1e-3) / 1e12 if self.gemm_ms > 0 else None
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(self.args.workload, {}).get("grouped_dgemm_bytes_per_launch")
        except OSError:
            pass
        kname = ("grouped_dgemm_tma<FUSED> (level-L formation + leaf products on DMMA mma.sync.m8n8k4.f64 + "
                 "level-L assembly, one persistent launch)" if self.fused else
                 "grouped_dgemm_tma (leaf products, mma.sync.m8n8k4.f64 = DMMA)")
        return {"bound": "tensor", "kernel": kname,
                "achieved": gemm_tf, "peak": self.dmma_peak, "unit": "TFLOP/s",
                "frac": (gemm_tf / self.dmma_peak) if gemm_tf else None, "traffic": traffic,
                "peak_source": "in-run DMMA microbenchmark fmm_probe_fp64_peak (MEASURED_PEAKS.json has no FP64 "
                               "figure; nameplate 148 SM x 128 flop/clk x 1.965 GHz = 37.2)",
                "algorithmic_flops_per_launch": st["leaf_flops"],
                "hidden_addition_bytes_per_launch": st["fused_add_bytes"]}

    def cpu_baseline(self):
        if self.rank != 0 or self.world != 1 or self.args.no_cpu:
            return None
        from oracle import oracle as O
        O.build()
        cpu = cpu_oracle_sample(self.w, self.A_np, self.B_np, self.args.cpu_frac)
        cpu.pop("seconds", None)
        return cpu

    # ---- the whole run -------------------------------------------------------------------------
    def sub_record(self, name, hbm, steps):
        """One extra BASELINE config on this GPU (N = 1), its own inputs and plan (configured algorithm
        and L, default options): effective GFLOPS over whole-step events (plain fmm_execute, graph replay
        where it applies), the leaf-GEMM fraction of the DMMA peak, the addition kernels' fraction of
        HBM (peel strips reported separately), cuBLAS on the same inputs, a sampled result check."""
        import numpy as np
        torch, F, stream = self.torch, self.F, self.stream
        w = WORKLOADS[name]
        P, Q, N, L = w["P"], w["Q"], w["N"], w["L"]
        flops = 2.0 * P * Q * N
        A_np, B_np = gen_inputs(w)
        A, B = to_device(A_np, w["layout"], self.device), to_device(B_np, w["layout"], self.device)
        del A_np, B_np
        alg = F.load_alg(w["alg"])
        plan = F.Plan(alg, P, Q, N, L, layout=w["layout"])
        st = plan.stats()
        C = plan.new_output()
        for _ in range(3):
            plan.execute(A, B, C, stream=stream)
        torch.cuda.synchronize()
        # launch-bound configs (c1: ~10 us per step) are timed over 200 calls, best of 3 passes,
        # like cuBLAS below, so the per-call host overhead and the event resolution average out
        small = flops < 1e9
        nrep = max(steps, 200) if small else steps
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = None
        for _ in range(3 if small else 1):
            e0.record(stream)
            for _ in range(nrep):
                plan.execute(A, B, C, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = min(ms or 1e30, e0.elapsed_time(e1) / nrep)
        plan.execute_timed(A, B, C, stream=stream)  # untimed: the first per-launch-event pass
        ph = np.median(np.array([[t["formation_ms"], t["gemm_ms"], t["assembly_ms"], t["strips_ms"], t["total_ms"]]
                                 for t in (plan.execute_timed(A, B, C, stream=stream)[1] for _ in range(5))]), axis=0)
        form_ms, gemm_ms, asm_ms, strip_ms, tot_ms = (float(x) for x in ph)
        # sampled rows (columns) of C against cuBLAS on the same rows, then cuBLAS on the whole problem
        g = torch.Generator().manual_seed(7)
        outer = P if w["layout"] == "row" else N
        idx = torch.randint(0, outer, (min(32, outer),), generator=g).to(self.device)
        err = ((C[idx] - A[idx] @ B) if w["layout"] == "row" else (C[:, idx] - A @ B[:, idx])).abs().max().item()
        tol = 1e-10 * torch.linalg.norm(A).item() * torch.linalg.norm(B).item()
        # cuBLAS timed like the plan above: `steps` back-to-back calls between two events (best of 2)
        cub = None
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Cc = torch.matmul(A, B)
        torch.cuda.synchronize()
        reps = nrep if small else steps if flops < 1e12 else 2
        for _ in range(3 if small else 2):
            c0.record()
            for _ in range(reps):
                torch.matmul(A, B, out=Cc)
            c1.record()
            c1.synchronize()
            cub = min(cub or 1e30, c0.elapsed_time(c1) / reps)
        del Cc
        add_bytes = st["add_bytes"] - st["fused_add_bytes"]
        leaf_tf = st["leaf_flops"] / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(name, {}).get("grouped_dgemm_bytes_per_launch")
        except OSError:
            pass
        rec = {"workload": w["desc"], "algorithm": w["alg"], "rank": alg.R, "levels": L, "P": P, "Q": Q, "N": N,
               "layout": w["layout"], "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOPS", "ms_per_step": ms,
               "steps": nrep, "warmup": 3,
               "timing": "CUDA events around the steps (plain fmm_execute)" + (", best of 3 passes" if small else ""),
               "effective_frac_of_fp64_peak": flops / (ms * 1e-3) / 1e12 / self.dmma_peak,
               "phases_ms": {"formation": form_ms, "leaf_gemm": gemm_ms, "assembly": asm_ms, "peel_strips": strip_ms,
                             "sum_of_launches_timed": tot_ms},
               "leaf_gemm": {"achieved_tflops": leaf_tf, "peak_tflops": self.dmma_peak,
                             "frac": (leaf_tf / self.dmma_peak) if leaf_tf else None,
                             "algorithmic_flops": st["leaf_flops"], "traffic_bytes_ncu": traffic},
               "additions": {"algorithmic_bytes": add_bytes, "ms": form_ms + asm_ms,
                             "gbs": add_bytes / ((form_ms + asm_ms) * 1e-3) / 1e9 if form_ms + asm_ms > 0 else None,
                             "frac_of_hbm": (add_bytes / ((form_ms + asm_ms) * 1e-3) / 1e9 / hbm)
                             if form_ms + asm_ms > 0 else None},
               "cublas_dgemm_gflops_same_inputs": flops / (cub * 1e-3) / 1e9 if cub else None,
               "vs_cublas": (cub / ms) if cub else None,
               "gpu_launches_per_step": int(st["launches"]),
               "collapsed_levels": bool(st.get("collapsed", 0)),
               "result_check": {"sampled": int(idx.numel()), "max_abs_err": err, "tolerance": tol, "ok": bool(err <= tol)}}
        del plan, A, B, C
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        return rec

    def go(self):
        args, w, st, world = self.args, self.w, None, self.world
        self.setup()
        st = self.st
        self.timed_steps()
        check = self.result_check()
        self.phase_split()
        add_ms = self.form_ms + self.asm_ms
        peaks, peak_src = measured_peaks()
        hbm = float(peaks.get("hbm_gbs", HBM_FALLBACK))
        sep_bytes = st["add_bytes"] - st["fused_add_bytes"]
        add_gbs = sep_bytes / (add_ms * 1e-3) / 1e9 if add_ms > 0 else None
        other = self.other_schedule()
        shape_matched = self.shape_matched()
        roofline = self.roofline()
        cub = self.cublas()
        own = self.own_classical()
        shards = self.shard_scaling()
        e2e = self.e2e()
        try:
            bcast = self.broadcast()
        except Exception as ex:  # noqa: BLE001  (measured after the timed region; must not cost the line)
            bcast = {"error": str(ex)[:300]}
        cpu = self.cpu_baseline()
        P, Q, N, ms_step, value = self.P, self.Q, self.N, self.ms_step, self.value
        names = args.configs
        if names == "auto":
            names = "c1,c3,c4,c5t,c5" if (world == 1 and args.workload == "c2") else "none"
        subs = None
        if names != "none" and world == 1:
            # the headline's buffers go first: c5's plan needs ~72 GB of the 180
            del self.plan
            self.A = self.B = self.C = None
            self.torch.cuda.synchronize()
            self.torch.cuda.empty_cache()
            subs = {}
            for nm in [x.strip() for x in names.split(",") if x.strip()]:
                try:
                    subs[nm] = self.sub_record(nm, hbm, max(3, min(args.steps, 10)))
                except Exception as ex:  # noqa: BLE001  (a sub-record must not cost the headline line)
                    subs[nm] = {"error": str(ex)[:300]}
                    self.torch.cuda.synchronize()
                    self.torch.cuda.empty_cache()
        if self.rank == 0:
            gb = lambda rows, cols: 8.0 * rows * cols / 1e9  # noqa: E731
            l2 = (f"inputs larger than L2 (A {gb(P, Q):.2f} GB, B {gb(Q, N):.2f} GB, C {gb(P, N):.2f} GB vs 126 MB); "
                  "no flush" if args.workload != "c1" else "small config: L2-resident")
            where = "reduce to rank 0" if args.output == "root" else "slab-distributed output"
            if world == 1:
                parallelism = "1 GPU"
            elif self.slab:
                parallelism = (f"slabs x{world}: every rank runs the whole method on its slab of C's "
                               f"{'rows' if w['layout'] == 'row' else 'columns'}; no partial products, no combine")
            elif args.combine == "p2p" or (args.combine == "p2p_push" and args.output == "slabs"):
                parallelism = (f"{args.shard_mode}-level shards x{world} + peer-memory combine inside fmm_execute "
                               f"(fmm_plan_create_p2p: one pull-reduce kernel per rank over CUDA IPC), {where}")
            elif args.combine == "p2p_push":
                parallelism = (f"{args.shard_mode}-level shards x{world} + peer-memory combine inside fmm_execute "
                               "(fmm_plan_create_p2p, p2p_push: the kernels that write C store each rank's partial "
                               "into rank 0's slots over CUDA IPC; rank 0 sums them), reduce to rank 0")
            elif args.combine == "lib":
                parallelism = (f"{args.shard_mode}-level shards x{world} + NCCL {where} inside fmm_execute "
                               "(fmm_plan_create_dist; C reduced in row chunks that overlap the assembly where the plan allows)")
            else:
                parallelism = f"{args.shard_mode}-level shards x{world} + {args.dist_backend.upper()} {where} (torch.distributed)"
            line = {
                "metric": METRIC, "value": value, "unit": "GFLOPS", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": w["desc"], "algorithm": w["alg"], "rank": self.alg.R, "levels": self.L,
                           "P": P, "Q": Q, "N": N, "layout": w["layout"],
                           "inputs": "uniform[-1,1) fp64, numpy PCG64 seeds 0 (A), 1 (B)",
                           "strategy": args.strategy, "cse": bool(args.cse), "l2": l2, "parallelism": parallelism,
                           "fused_leaf_level": self.fused, "collapsed_levels": bool(st.get("collapsed", 0)),
                           **({"dist_backend": "gloo (control-flow check, ranks share a GPU: NOT a measurement)"}
                              if world > 1 and args.dist_backend == "gloo" else {})},
                "roofline": roofline,
                "clocks": self.clk,
                "e2e": e2e,
                "gpu_launches": (int(st["launches"]) + (1 if args.combine in ("p2p", "p2p_push") and world > 1 else 0))
                * args.steps,
                "cpu_baseline": cpu,
                "phases_ms": {"formation_levels_below_L" if self.fused else "formation": self.form_ms,
                              "fused_leaf_level" if self.fused else "leaf_gemm": self.gemm_ms,
                              "assembly": self.asm_ms, "peel_strips": self.strip_ms,
                              "combine_exposed": self.comm_ms if world > 1 else 0.0,
                              "how": "fmm_execute_timed after the timed steps: plain launches, an event after each, "
                                     "median of 5 after an untimed pass"},
                "input_broadcast": bcast,
                "combine_algbw_gbs": (8.0 * P * N / (self.comm_ms * 1e-3) / 1e9) if world > 1 and self.comm_ms else None,
                "additions": {"algorithmic_bytes_per_step": st["add_bytes"],
                              "bytes_in_fused_launch": st["fused_add_bytes"],
                              "separate_kernel_bytes": sep_bytes, "separate_kernel_gbs": add_gbs, "peak_gbs": hbm,
                              "separate_kernel_frac": (add_gbs / hbm) if add_gbs else None, "peak_source": peak_src},
                "other_schedule": other,
                "shape_matched": shape_matched,
                "fp64_peak_tflops": {"dmma_measured": self.dmma_peak, "dfma_measured": self.dfma_peak, "nameplate": 37.2},
                "effective_frac_of_fp64_peak": value / 1e3 / self.dmma_peak,
                "cublas_dgemm_gflops_same_inputs": cub,
                "classical_own_dgemm": own,
                "result_check": check,
                "paper_effective_gflops": (2.0 * P * Q * N - P * N) / (ms_step * 1e-3) / 1e9,
                "plan": {k: st[k] for k in ("gemm_flops", "add_flops", "add_bytes", "launches", "leaves")},
                "configs": subs,
                "shard_compute_scaling": shards,
            }
            print(json.dumps(line), flush=True)
        if world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


if __name__ == "__main__":
    main()
