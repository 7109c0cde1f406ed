"""Summarises an ncu `--page source --csv` (SASS view) export: warp-level
instructions executed and stall samples per SASS mnemonic, top stalled
instructions."""
import csv
import sys
from collections import defaultdict


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    print(f"source: {path}  {rows[0][1][:80]}")
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    by_op = defaultdict(lambda: [0.0, 0.0])
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ins = num(r[ix["Instructions Executed"]])
        smp = num(r[ix["Warp Stall Sampling (All Samples)"]])
        by_op[op][0] += ins
        by_op[op][1] += smp
        recs.append((smp, ins, r[ix["Address"]], src))
    ti = sum(v[0] for v in by_op.values())
    ts = sum(v[1] for v in by_op.values())
    print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
    print("  op           instr%   stall%")
    for op, (i, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {op:12s} {100 * i / ti:6.2f}  {100 * s / ts:6.2f}")
    print("top stalled instructions:")
    for smp, ins, addr, src in sorted(recs, reverse=True)[:15]:
        print(f"  {100 * smp / ts:5.2f}%  {addr}  {src[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
