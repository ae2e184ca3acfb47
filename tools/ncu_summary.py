"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per kernel family -> launches, total us, share of the listed device time."""
import collections
import csv
import json
import re
import sys


def family(name):
    name = name.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    n = re.sub(r"[<(].*", "", name).replace("void ", "").strip()
    m = re.search(r"<([^>]*)>\(", name)
    args = [a.strip().replace("(bool)", "").replace("(int)", "") for a in m.group(1).split(",")] if m else []
    if args and n.endswith(("tile_conv_kernel", "tile_conv_kernel_capped")):
        # <FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, JT, SPARSE, EPI>
        sparse = args[11] if len(args) > 12 else args[-1]
        jt = args[10] if len(args) > 10 else "0"
        kind = "[jump-table]" if jt == "100" else "[counted-dense]" if jt == "200" else ""
        n += ("<FWD>" if args[0] in ("1", "true") else "<BWI>") + ("[sparse]" if sparse in ("1", "true") else "[dense]")
        n += kind
    elif args and n.endswith("bww_tile_kernel"):
        n += ("<check=input>" if args[0] in ("1", "true") else "<check=output_grad>")
        n += "[sparse]" if args[-1] in ("1", "true") else "[dense]"
    return n


# setup-only kernels of tools/one_step.py (synthetic data, packing, the BWW
# operand's ActCHWNn copy): not part of the timed bench step
SETUP = ("at::", "nchwc_to_chwnn")


def main(path, out_json=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        us = v / 1000.0 if unit in ("ns", "nsecond") else v * 1000.0 if unit in ("ms", "msecond") else v
        f = family(r[ik])
        if any(f.startswith(x) or x in f for x in SETUP):
            continue
        agg[f][0] += 1
        agg[f][1] += us
    tot = sum(v[1] for v in agg.values())
    res = {k: {"launches": v[0], "total_us": round(v[1], 1), "share": round(v[1] / tot, 4)}
           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
    for k, v in res.items():
        print(f"{v['share']*100:6.2f}%  {v['total_us']:12.1f} us  {v['launches']:5d}  {k}")
    if out_json:
        json.dump({"source": path, "note": "one bench step (tools/one_step.py) under ncu --metrics gpu__time_duration.sum "
                   "--clock-control none; setup kernels excluded; per-launch times are cold-cache and serialised",
                   "total_us": round(tot, 1), "kernels": res}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
