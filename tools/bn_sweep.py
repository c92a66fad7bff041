"""Leaf-GEMM tile width sweep per BASELINE workload (FMM_GEMM_BN), default plan options."""
import os, subprocess, sys
for cfg in sys.argv[1:]:
    for bn in ["auto", "128", "112", "96", "80", "64"]:
        env = dict(os.environ)
        if bn != "auto":
            env["FMM_GEMM_BN"] = bn
        out = subprocess.run([sys.executable, "tools/collapse_timing.py", cfg], env=env, capture_output=True, text=True).stdout
        line = [l for l in out.splitlines() if l.startswith(cfg)]
        print(cfg, "BN", bn, line[0].split("|")[1].strip() if line else out[-300:], flush=True)
