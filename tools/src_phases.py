#!/usr/bin/env python3
"""Stall samples of an ncu `--page source --csv` export in program order:
prints every SASS row holding >= thr% of the samples, with the running share
and the executed count (to see which phase of a kernel stalls)."""
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main(path, thr=0.4):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    recs = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        recs.append((r[ix["Source"]].strip(), num(r[ix["Warp Stall Sampling (All Samples)"]]),
                     num(r[ix["Instructions Executed"]]),
                     {k[6:]: num(r[ix[k]]) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}))
    tot = sum(r[1] for r in recs)
    toti = sum(r[2] for r in recs)
    print(f"{path}: {len(recs)} SASS rows, {tot:.0f} samples, {toti:.3e} warp instr")
    run = 0.0
    runi = 0.0
    for i, (src, smp, ins, st) in enumerate(recs):
        run += smp
        runi += ins
        if smp >= thr / 100 * tot:
            top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
            tops = " ".join(f"{k}:{100 * v / max(smp, 1):.0f}%" for k, v in top)
            print(f"{i:5d} {100 * smp / tot:5.2f}% cum {100 * run / tot:5.1f}% (instr cum {100 * runi / toti:5.1f}%) x{ins:.2e}  {src[:60]:60s} {tops}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.4)
