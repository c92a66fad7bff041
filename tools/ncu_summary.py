"""Summarise an ncu --set full report (per kernel: time, DRAM bytes, pipe utilisation, stalls)
into JSON + Markdown under profiles/.  Usage: python tools/ncu_summary.py REP.ncu-rep OUT_PREFIX"""
import csv, io, json, subprocess, sys

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read_GB": "dram__bytes_read.sum",
    "dram_write_GB": "dram__bytes_write.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block_KB": "launch__shared_mem_per_block",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "shared_excessive_wavefronts": "derived__memory_l1_wavefronts_shared_excessive",
}
UNIT_SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3,
              "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:80]}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if k.endswith("_GB") or k == "time_ms":
                    v *= UNIT_SCALE.get(u, 1.0)
                d[k] = v
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        d["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        kernels.append(d)
    json.dump({"report": rep, "kernels": kernels}, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu --set full summary of `{rep}`\n\n")
        f.write("| kernel | time ms | DRAM rd GB | DRAM wr GB | tensor pipe % | DRAM % | regs | grid x block | top stalls (% of samples) |\n|---|---|---|---|---|---|---|---|---|\n")
        for d in kernels:
            f.write(f"| {d['kernel'][:40]} | {d.get('time_ms', 0):.3f} | {d.get('dram_read_GB', 0):.3f} | {d.get('dram_write_GB', 0):.3f} | "
                    f"{d.get('tensor_pipe_pct', 0):.1f} | {d.get('dram_throughput_pct', 0):.1f} | {d.get('registers', 0):.0f} | "
                    f"{d.get('grid', 0):.0f} x {d.get('block', 0):.0f} | "
                    + ", ".join(f"{k} {v}" for k, v in d["top_stalls_pct"].items()) + " |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
