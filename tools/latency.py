#!/usr/bin/env python3
"""Single-image lola-mnist HE-step latency (29-bit set), with and without
CUDA-graph replay, for A/B runs (LB_KS_PAIR / LB_NTT_PAIR / LB_LIB): one JSON line."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    cx = BfvContext(lola_mnist_params_w32())
    net = nets.lola_mnist_net(config=2)
    imgs = nets.images(2, net, B)
    one = Session(cx, net, "lola-mnist", B)
    dev = torch.from_numpy(imgs.copy()).cuda()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    for graph in (False, True):
        if graph:
            one.set_graph(True)
        one.encrypt(dev, on_device=True)
        for _ in range(3):
            one.execute()
        torch.cuda.synchronize()
        lat = []
        for _ in range(7):
            e0.record(s)
            one.execute()
            e1.record(s)
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1))
        out["graph" if graph else "no_graph"] = round(min(lat), 3)
    print(json.dumps({"images": B, "he_steps_ms": out}))


if __name__ == "__main__":
    main()
