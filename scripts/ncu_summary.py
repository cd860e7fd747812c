"""Summarise ncu --set full reports (scripts/ncu_capture.sh) into one JSON:
duration, SM / DRAM throughput, occupancy, registers, DRAM bytes, FP64 and
DMMA pipe utilisation, and the top warp-stall reasons (PC sampling).
Usage: python scripts/ncu_summary.py out.json gpurun_out/ncu_*.ncu-rep"""
import csv, io, json, subprocess, sys

KEYS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # ncu units -> ns, then us
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_throughput_pct": ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "grid_size": ("launch__grid_size", 1),
    "block_size": ("launch__block_size", 1),
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "dmma_pipe_pct": ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    s = {"report": rep.split("/")[-1], "kernel": vals[col["Kernel Name"]][:120]}
    for k, (m, sc) in KEYS.items():
        if m in col:
            try:
                v = float(vals[col[m]].replace(",", ""))
                v *= UNIT.get(units[col[m]], 1)
                s[k] = v * sc
            except ValueError:
                pass
    stalls = {}
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    s["top_stalls_share"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
    return s


res = [summarise(r) for r in sys.argv[2:]]
json.dump(res, open(sys.argv[1], "w"), indent=1)
for r in res:
    print(json.dumps(r))
