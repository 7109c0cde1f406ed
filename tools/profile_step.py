#!/usr/bin/env python3
"""One lola-mnist HE step (the bench's unit of work) bracketed by
cudaProfilerStart/Stop, for `ncu --profile-from-start off`: the launch list
and the full captures then cover exactly one step after warm-up."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--workload", default="lola-mnist")
    ap.add_argument("--word", type=int, default=32)
    a = ap.parse_args()
    import torch

    import bench
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session

    cfg, strategy, _, net, prm = bench.workload_objects(a.workload, a.word)
    cx = BfvContext(prm)
    sess = Session(cx, net, strategy, a.batch)
    imgs = torch.from_numpy(nets.images(cfg, net, a.batch)).cuda()
    sess.encrypt(imgs, on_device=True)
    sess.execute()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    sess.execute()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one step:", a.workload, "batch", a.batch)


if __name__ == "__main__":
    main()
