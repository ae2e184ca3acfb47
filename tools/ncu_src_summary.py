"""Summarise an `ncu --page source --csv --print-source sass` log: stall
samples by SASS opcode class and the hottest instructions."""
import collections
import csv
import io
import sys


def load(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    kern = rows[0][1] if len(rows[0]) > 1 else rows[0][0]
    hdr = rows[1]
    return kern, hdr, rows[2:]


def main(path, top=30):
    kern, hdr, rows = load(path)
    iS, iN, iE, iSrc = (hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)"),
                        hdr.index("Instructions Executed"), hdr.index("Source"))
    by_op = collections.Counter()
    ex_op = collections.Counter()
    tot = 0
    recs = []
    for r in rows:
        try:
            s = float(r[iS] or 0)
            e = float(r[iE] or 0)
        except ValueError:
            continue
        src = r[iSrc].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        by_op[op] += s
        ex_op[op] += e
        tot += s
        recs.append((s, e, src))
    print(kern[:150])
    print(f"total stall samples {tot:.0f}; instructions executed {sum(ex_op.values()):.3g}")
    for op, s in by_op.most_common(15):
        print(f"  {op:10s} samples {100 * s / tot:5.1f}%   executed {100 * ex_op[op] / sum(ex_op.values()):5.1f}%")
    print("hottest instructions:")
    for s, e, src in sorted(recs, reverse=True)[:top]:
        print(f"  {100 * s / tot:5.2f}%  exec {e:10.3g}  {src[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
