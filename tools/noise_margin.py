#!/usr/bin/env python3
"""Noise margin of a lola-mnist parameter set, measured on the device
ciphertexts: run the plan on a few images, then for every output message and
plaintext instance j compute the phase x = c0 + c1 s (CPU oracle, exact) and
the invariant noise |[t_j x]_Q| (centered). Decryption is correct while it
stays below Q/2; margin = log2(Q/2) - log2(max |[t x]_Q|) bits. Also checks
the decrypted logits against forward_integer and times one batched step.

usage: python tools/noise_margin.py L K dnum bits [batch] [workload]
(workload lola-mnist: n = 16384, 5 plaintext primes; lola-small: n = 8192, 2;
lola-cifar: n = 16384, 6)"""
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    L, K, dnum, bits = (int(v) for v in sys.argv[1:5])
    batch = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    workload = sys.argv[6] if len(sys.argv) > 6 else "lola-mnist"
    import numpy as np
    import torch

    from oracle import bfvbind as O
    from oracle import refbind as R
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session
    from paper_1812_10659_b200.params import make_params

    n, T, cfg = {"lola-mnist": (16384, 5, 2), "lola-small": (8192, 2, 3), "lola-cifar": (16384, 6, 4)}[workload]
    prm = make_params(n, L=L, T=T, K=K, dnum=dnum, bits=bits)
    print(f"L={L} K={K} dnum={dnum} bits={bits}: log2 QP = {prm.log_qp():.1f}, log2 Q = "
          f"{sum(math.log2(v) for v in prm.q):.1f}", flush=True)
    cx = BfvContext(prm)
    net = {"lola-mnist": lambda: nets.lola_mnist_net(config=2), "lola-small": lambda: nets.lola_small_net(config=3),
           "lola-cifar": lambda: nets.lola_cifar_net(config=4)}[workload]()
    sess = Session(cx, net, workload, batch)
    imgs = nets.images(cfg, net, batch)
    scores, _, _ = sess.run(imgs)
    exact = all(scores[b] == R.forward_integer(net, imgs[b]) for b in range(batch))
    print("decrypted logits == forward_integer:", exact, flush=True)
    o = O.Oracle.from_params(prm)
    Q = math.prod(prm.q)
    coef = [(Q // qi) * pow(Q // qi, -1, qi) for qi in prm.q]
    worst = 0
    outs = 0
    while True:
        try:
            dev = sess.output_ciphertexts(outs)
            x = dev.reshape(-1, prm.L, prm.n).to(torch.int64)
            cx.ntt_inverse(x, limbs=prm.L)  # evaluation -> coefficient domain (the oracle's layout)
            torch.cuda.synchronize()
            cts = x.reshape(dev.shape).cpu().numpy().astype(np.uint64)
        except Exception:
            break
        outs += 1
        for j, t in enumerate(prm.t):
            x = o.phase(cts[0, j])
            cols = [x[i].tolist() for i in range(prm.L)]
            for k in range(prm.n):
                v = sum(cols[i][k] * coef[i] for i in range(prm.L)) % Q
                e = (t * v) % Q
                if e > Q // 2:
                    e -= Q
                worst = max(worst, abs(e))
        if outs >= 2:
            break
    print(f"outputs checked {outs}: max |[t x]_Q| = 2^{math.log2(worst):.1f}; margin "
          f"{math.log2(Q / 2) - math.log2(worst):.1f} bits", flush=True)
    del sess
    torch.cuda.empty_cache()
    B = {"lola-mnist": 64, "lola-small": 256, "lola-cifar": 1}[workload]
    sess = Session(cx, net, workload, B)
    sess.encrypt(torch.from_numpy(nets.images(cfg, net, B)).cuda(), on_device=True)
    reps = 1 if workload == "lola-cifar" else 3
    for _ in range(reps):
        sess.execute()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sess.execute()
    e1.record()
    torch.cuda.synchronize()
    print(f"throughput B={B}: {reps * B / (e0.elapsed_time(e1) / 1e3):.2f} images/s", flush=True)


if __name__ == "__main__":
    main()
