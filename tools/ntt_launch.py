#!/usr/bin/env python3
"""The hot-path NTT launches bench.py's roofline_ntt times (u32 residues,
n = 16384, the key switch's limb count at the bench batch), one forward and
one inverse after warm-up, bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off`."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    prm = lola_mnist_params_w32()
    cx = BfvContext(prm)
    limbs = 64 * 5 * prm.dnum * (prm.L + prm.K - 1)
    data = torch.randint(0, min(prm.q), (limbs // prm.L, prm.L, prm.n), dtype=torch.int32, device="cuda")
    for _ in range(3):
        cx.ntt_forward(data, limbs=prm.L)
        cx.ntt_inverse(data, limbs=prm.L)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    cx.ntt_forward(data, limbs=prm.L)
    cx.ntt_inverse(data, limbs=prm.L)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled", limbs, "limbs")


if __name__ == "__main__":
    main()
