#!/usr/bin/env python3
"""BASELINE config 1: HE primitive throughput on one B200.

Batches of 64 ciphertexts at n in {4096, 8192, 16384, 32768} and L ciphertext
limbs: NTT/INTT limb transforms per second (and Gbutterfly/s against the
measured integer roof), ct x pt, ct + ct, rotations (key switches) and
square + relinearize per second. Device-timed with CUDA events after warm-up;
inputs (64 x 2 x L x n x 8 B, >= 8 MiB per operand) stream through HBM.
Prints one JSON object per (n, L); `--out` also writes them to a file.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))


def timed(fn, reps):
    import torch

    s = torch.cuda.current_stream()
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    import torch

    from paper_1812_10659_b200 import _native as nat
    from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns
    from paper_1812_10659_b200.params import make_params

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--grid", default="4096:2,4096:6,8192:4,8192:8,16384:4,16384:6,16384:12,32768:4,32768:12")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    peak = C.c_double()
    lines = []
    for spec in a.grid.split(","):
        parts = [int(x) for x in spec.split(":")]
        n, L = parts[:2]
        K = parts[2] if len(parts) > 2 else 1
        dnum = parts[3] if len(parts) > 3 else L
        prm = make_params(n, L=L, T=1, K=K, dnum=dnum, seed=1)
        cx = BfvContext(prm)
        nat.call("lb_bench_butterfly_peak", prm.q[0], 4, 2000, C.byref(peak))
        B = a.batch
        vals = torch.randint(-1000, 1000, (B, n), dtype=torch.int64, device="cuda")
        ct = cx.encrypt_slots(vals, id_base=1)
        ct2 = cx.encrypt_slots(vals, id_base=B + 1)
        pm, _ = cx.encode_plain(vals[0], add=False)
        out = torch.empty_like(ct)
        limbs = torch.randint(0, 2**59, (B * 2, L, n), dtype=torch.int64, device="cuda")
        g = galois_exponent_columns(n, 1)
        cx.keygen(g)
        cx.keygen(0)
        t_fwd = timed(lambda: cx.ntt_forward(limbs, limbs=L), a.reps)
        t_inv = timed(lambda: cx.ntt_inverse(limbs, limbs=L), a.reps)
        t_mp = timed(lambda: cx.mul_plain(ct, pm, out=out), a.reps)
        t_add = timed(lambda: cx.add(ct, ct2, out=out), a.reps)
        t_rot = timed(lambda: cx.rotate(ct, g, out=out), max(2, a.reps // 2))
        t_sq = timed(lambda: cx.mul(ct, ct, out=out), max(2, a.reps // 2))
        nlimb = B * 2 * L
        bfly = nlimb * (n // 2) * (n.bit_length() - 1)
        ct_bytes = 2 * L * n * 8
        rec = {
            "n": n, "L": L, "batch": B, "K": K, "dnum": dnum,
            "ntt_fwd_limbs_per_s": nlimb / t_fwd, "ntt_inv_limbs_per_s": nlimb / t_inv,
            "ntt_fwd_gbfly_s": bfly / t_fwd / 1e9, "int_peak_gbfly_s": peak.value / 1e9,
            "ntt_fwd_frac_of_int_peak": bfly / t_fwd / peak.value,
            "ct_pt_per_s": B / t_mp, "ct_pt_gbs": B * (ct_bytes * 2 + L * n * 8) / t_mp / 1e9,
            "ct_add_per_s": B / t_add, "ct_add_gbs": B * ct_bytes * 3 / t_add / 1e9,
            "rotations_per_s": B / t_rot, "square_relin_per_s": B / t_sq,
        }
        lines.append(rec)
        print(json.dumps(rec), flush=True)
        del cx, ct, ct2, out, limbs
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text("\n".join(json.dumps(r) for r in lines) + "\n")


if __name__ == "__main__":
    main()
