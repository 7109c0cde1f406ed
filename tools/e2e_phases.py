#!/usr/bin/env python3
"""Wall-clock split of one end-to-end lola-mnist run (host pixels -> encode +
encrypt -> HE steps -> decrypt + CRT -> host logits) at the bench's batch:
where the e2e number loses against the device-resident `value`."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    import bench
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    cfg, strategy, _, net, prm = bench.workload_objects("lola-mnist", 32)
    cx = BfvContext(prm)
    from paper_1812_10659_b200 import _native as nat

    nat.call("lb_pool_reserve", cx.handle, int(torch.cuda.mem_get_info()[0] * 0.5))
    sess = Session(cx, net, strategy, B)
    imgs = np.ascontiguousarray(nets.images(cfg, net, B))
    scores = np.zeros((B, sess.outputs, 4), dtype=np.uint64)
    sess.run_raw(imgs, scores, False, False, want_counters=False, want_times=True)  # warm
    for _ in range(3):
        t0 = time.perf_counter()
        _, times = sess.run_raw(imgs, scores, False, False, want_counters=False, want_times=True)
        wall = time.perf_counter() - t0
        print(f"B={B}: encode+encrypt {times[0] * 1e3:.1f} ms, HE steps {times[1] * 1e3:.1f} ms, "
              f"decrypt+CRT {times[2] * 1e3:.1f} ms, wall {wall * 1e3:.1f} ms -> {B / wall:.1f} images/s")


if __name__ == "__main__":
    main()
