#!/usr/bin/env python3
"""One encrypt and one decrypt of a lola-mnist batch (bench batch), each
bracketed by cudaProfilerStart/Stop for `ncu --profile-from-start off`
launch lists: where the end-to-end path's non-HE time goes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    import bench
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session

    phase = sys.argv[1] if len(sys.argv) > 1 else "decrypt"
    B = 64
    cfg, strategy, _, net, prm = bench.workload_objects("lola-mnist", 32)
    cx = BfvContext(prm)
    sess = Session(cx, net, strategy, B)
    imgs = np.ascontiguousarray(nets.images(cfg, net, B))
    for _ in range(2):
        sess.encrypt(imgs)
        sess.execute()
        sess.decrypt()
    torch.cuda.synchronize()
    prof = torch.cuda.cudart()
    prof.cudaProfilerStart()
    if phase == "encrypt":
        sess.encrypt(imgs)
    else:
        sess.decrypt()
    torch.cuda.synchronize()
    prof.cudaProfilerStop()
    print("profiled", phase)


if __name__ == "__main__":
    main()
