#!/usr/bin/env python3
"""Key-switch and NTT rooflines alone (bench.py's formulas), for A/B runs of
variant builds (LB_LIB=<variant>): one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import bench
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    prm = lola_mnist_params_w32()
    cx = BfvContext(prm)
    cx.keygen(bench_galois(prm.n))
    import os
    ks = bench.ks_roofline(cx, int(os.environ.get("KB_COUNT", "320")))
    ntt = bench.ntt_roofline(cx, 64 * 5 * prm.dnum * (prm.L + prm.K - 1))
    print(json.dumps({"ks_frac": round(ks["frac"], 4), "ks_ms": round(ks["launch_set_ms"], 4),
                      "ntt_frac": round(ntt["frac"], 4), "ntt_fwd": round(ntt["frac_forward"], 4),
                      "ntt_inv": round(ntt["frac_inverse"], 4), "peak": round(ks["peak"], 1)}))


def bench_galois(n):
    from paper_1812_10659_b200.bfv import galois_exponent_columns

    return galois_exponent_columns(n, 1)


if __name__ == "__main__":
    main()
