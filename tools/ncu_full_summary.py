"""Extract the judged metrics from `ncu --set full` captures into JSON:
duration, DRAM bytes (traffic), FP32-pipe utilisation, issue activity,
occupancy, L1/L2 throughput and the warp-stall mix."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cycles_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def summarize(rep):
    """`rep`: an .ncu-rep, or the CSV log of `ncu --set full --csv --page raw
    --log-file X` (the form this pool's ncu wrapper returns intact)."""
    if rep.endswith(".csv"):
        raw = "".join(ln for ln in open(rep) if ln.startswith('"'))
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    return [summarize_row(rep, hdr, units, vals) for vals in rows[2:]]


def summarize_row(rep, hdr, units, vals):
    out = {"report": rep.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")][:160]}
    stalls = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e-6, "msecond": 1e-3,
                     "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(u, 1)
            out[KEYS[h]] = f * scale if u in ("Kbyte", "Mbyte", "Gbyte", "byte") else f
            if h == "gpu__time_duration.sum":
                out["duration_s"] = f * scale
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                n = float(v.replace(",", ""))
            except ValueError:
                continue
            if n:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = n
    tot = sum(stalls.values()) or 1
    out["stall_mix_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])}
    out["dram_bytes"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    return out


if __name__ == "__main__":
    res = [r for p in sys.argv[2:] for r in summarize(p)]
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    for r in res:
        print(json.dumps({k: r[k] for k in r if k != "stall_mix_pct"}))
        print("   stalls:", r["stall_mix_pct"])
