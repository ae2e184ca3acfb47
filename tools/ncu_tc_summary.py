"""Summarise `ncu --set full` captures of the tensor-core (tcgen05) kernels:
duration, tensor-pipe activity, L2 / TMA / DRAM throughput, DRAM bytes,
registers, grid, SM clock.  Usage: ncu_tc_summary.py out.json rep1 [rep2 ...]"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.pct_of_peak_sustained_elapsed": "tma_load_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "dram__bytes_read.sum": "dram_read_mb",
    "dram__bytes_write.sum": "dram_write_mb",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_ghz",
}


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if "tc_" not in name:
            continue
        d = {"kernel": name.split("(")[0].replace("void ", "").replace("unnamed>::", "")}
        for k, v in KEYS.items():
            if k in h:
                try:
                    d[v] = round(float(r[h.index(k)]), 3)
                except ValueError:
                    d[v] = r[h.index(k)]
        out.append(d)
    return out


if __name__ == "__main__":
    res = {"note": "ncu --set full --clock-control none, VGG16 conv3_2 (N=32, C=K=256, 56x56, 3x3 s1), s=0.6, "
                   "spc_set_math(SPC_MATH_TF32X3); tensor_pipe_active_pct = "
                   "sm__pipe_tensor_subpipe_hmma_cycles_active (pct of peak sustained active)",
           "captures": {}}
    for rep in sys.argv[2:]:
        res["captures"][rep.split("/")[-1]] = summarize(rep)
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])
