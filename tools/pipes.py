#!/usr/bin/env python3
"""Integer-pipe cross-check of the butterfly roof: thread-level
issue rates of IMAD, IMAD.HI, IADD3 and the conditional subtraction, next to
the register-resident Shoup butterfly rate, on the current GPU."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1812_10659_b200 import _native as nat

    torch.cuda.init()
    ops = (C.c_double * 5)()
    nat.call("lb_bench_int_pipes", 20000, ops)
    peak32, peak64 = C.c_double(), C.c_double()
    nat.call("lb_bench_butterfly_peak", 536608769, 4, 4000, C.byref(peak32))
    nat.call("lb_bench_butterfly_peak", 1152921504606584833, 4, 4000, C.byref(peak64))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    out = {"imad_gops": ops[0] / 1e9, "imad_hi_gops": ops[1] / 1e9, "iadd3_gops": ops[2] / 1e9,
           "lop3_viaddmnmx_pairs_gops": ops[3] / 1e9, "imad_wide_gops": ops[4] / 1e9, "butterfly32_gbfly_s": peak32.value / 1e9,
           "butterfly64_gbfly_s": peak64.value / 1e9, "sms": sms}
    # FMA-pipe bound of one 32-bit Shoup butterfly: IMAD.HI + 2 IMAD
    out["butterfly32_fma_pipe_bound_gbfly_s"] = 1.0 / (1.0 / out["imad_hi_gops"] + 2.0 / out["imad_gops"])
    out["butterfly32_frac_of_fma_bound"] = out["butterfly32_gbfly_s"] / out["butterfly32_fma_pipe_bound_gbfly_s"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
