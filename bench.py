#!/usr/bin/env python3
"""LoLa-MNIST encrypted inference throughput on B200 (BASELINE.json config 2).

One step = one pass of the HE hot path (the lola-mnist plan at n = 16384,
5 plaintext-prime BFV instances per image) over a batch of encrypted images
already resident in HBM. Multi-GPU: one process per GPU (torchrun), images
sharded across ranks with no collective on the data path;
NCCL only for the barrier and the max-over-ranks timing.

`--impl reference` times the reference's own CPU implementation (packnn,
compiled in place into oracle/_ref/libpackref.so) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "LoLa-MNIST encrypted inferences/s & latency; NTT/s, rotations/s vs roofline"
UNIT = "inferences/s"

# workload -> (BASELINE config, strategy, default images per GPU per step)
WORKLOADS = {
    "lola-mnist": (2, "lola-mnist", 64),
    "lola-small": (3, "lola-small", 256),
    "lola-cifar": (4, "lola-cifar", 1),
    # the CryptoNets baseline representation of the paper's comparison: the
    # cfg0 net with one message per value and the images in the slots
    # (n = 16384 images per step); not a BASELINE config
    "cryptonets-simd": (2, "cryptonets-simd", 16384),
}


def workload_objects(name: str, word: int = 64):
    from paper_1812_10659_b200 import nets, params

    cfg, strategy, batch = WORKLOADS[name]
    if name == "lola-mnist":
        prm = params.lola_mnist_params_w32() if word == 32 else params.lola_mnist_params()
        return cfg, strategy, batch, nets.lola_mnist_net(config=2), prm
    if name == "cryptonets-simd":
        prm = params.lola_mnist_params_w32() if word == 32 else params.lola_mnist_params()
        return cfg, strategy, batch, nets.lola_mnist_net(config=2), prm
    if name == "lola-small":
        prm = params.lola_small_params_w32() if word == 32 else params.lola_small_params()
        return cfg, strategy, batch, nets.lola_small_net(config=3), prm
    prm = params.lola_cifar_params_w32() if word == 32 else params.lola_cifar_params()
    return cfg, strategy, batch, nets.lola_cifar_net(config=4), prm


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=0, help="images per GPU per step (default per workload)")
    ap.add_argument("--workload", default="lola-mnist", choices=list(WORKLOADS),
                    help="lola-mnist = BASELINE config 2 (the headline); lola-small = config 3; lola-cifar = config 4; "
                         "cryptonets-simd = the cfg0 net in the CryptoNets representation (images in slots)")
    ap.add_argument("--cpu-sample", type=int, default=6, help="images in the single-thread CPU baseline sample")
    ap.add_argument("--no-extras", action="store_true", help="skip latency / roofline / CPU baseline legs")
    ap.add_argument("--word", type=int, default=32, choices=[32, 64],
                    help="RNS word: 32 = 29/30-bit primes (32-bit word kernels, u32 residues; default), "
                         "64 = 54/60-bit primes")
    return ap.parse_args()


# ---- distributed plumbing -----------------------------------------------------------

def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    from paper_1812_10659_b200.shard import barrier as _b

    _b(world)


def max_over_ranks(world, value: float) -> float:
    from paper_1812_10659_b200.shard import max_over_ranks as _m

    return _m(value, world, device="cuda")


# ---- clocks ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        if os.environ.get("LB_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's NVML start-up must not overlap the timed region
            t0 = time.time()
            while not self.lines and time.time() - t0 < 10:
                time.sleep(0.05)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons, power = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(name)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "sm_min_mhz": sm[0] if sm else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ---- CPU baseline (reference) ---------------------------------------------------------

def _ref_worker(args):
    idx_list, = args
    from oracle import refbind as R
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.params import lola_mnist_params

    net = nets.lola_mnist_net()
    prm = lola_mnist_params()
    tot = 0.0
    for i in idx_list:
        x = nets.images(2, net, 1, start=i)[0]
        enc, steps = R.time_plan_steps(net, "lola-mnist", prm.n, prm.t, x, ring=True, threads=1)
        tot += enc + float(steps.sum())
    return tot


def cpu_reference_throughput(images: int, procs: int) -> tuple[float, float]:
    """Reference ring backend, encode + HE steps per image (decode excluded),
    `procs` independent single-thread processes; returns (images/s, wall s)."""
    import multiprocessing as mp

    per = [list(range(p, images, procs)) for p in range(procs)]
    per = [p for p in per if p]
    t0 = time.perf_counter()
    if len(per) == 1:
        _ref_worker((per[0],))
    else:
        with mp.get_context("spawn").Pool(len(per)) as pool:
            pool.map(_ref_worker, [(p,) for p in per])
    wall = time.perf_counter() - t0
    return images / wall, wall


# ---- reference arm ----------------------------------------------------------------------

def run_reference(a, world, rank):
    if rank != 0:
        return
    from oracle import refbind as R

    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpackref.so not built"}))
        return
    cores = os.cpu_count() or 1
    for _ in range(a.warmup):
        cpu_reference_throughput(cores, cores)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        cpu_reference_throughput(cores, cores)
    wall = time.perf_counter() - t0
    value = a.steps * cores / wall
    sample = (f"{cores} images per step (one per process, {cores} single-thread processes); "
              "lola-mnist n=16384, 5 plaintext primes, ring backend, encode + HE steps (decode excluded: "
              "the Boost stand-in BigInt is not representative)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": wall / a.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "lola-mnist cfg2 batched throughput (reference packnn ring backend, CPU)",
                   "images_per_step": cores, "n": 16384, "plain_primes": 5},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---- our arm -----------------------------------------------------------------------------

TRAFFIC_JSON = ROOT / "profiles" / "ncu_traffic.json"


def ncu_traffic(match) -> tuple[float | None, str | None]:
    """DRAM bytes per unit (ciphertext or limb) summed over the committed ncu
    --set full captures whose kernel name satisfies `match` (written by
    profiles/traffic_from_ncu.py); (None, None) when absent."""
    try:
        d = json.loads(TRAFFIC_JSON.read_text())
    except Exception:
        return None, None
    ks = {k: v for k, v in d["kernels"].items() if match(k)}
    if not ks:
        return None, None
    return sum(v["bytes_per_unit"] for v in ks.values()), f"{TRAFFIC_JSON.relative_to(ROOT)}: " + ", ".join(sorted(ks))


def ntt_roofline(cx, limbs: int, reps: int = 20) -> dict:
    """Dominant kernel (batched NTT at n=16384, the workload's word size)
    timed alone with CUDA events on its launch stream, against the measured
    integer-pipe roof of the same word size."""
    import ctypes as C

    import torch

    from paper_1812_10659_b200 import _native as nat

    n, L = cx.n, cx.L
    polys = max(1, limbs // L)
    data = torch.randint(0, min(cx.params.q), (polys, L, n), dtype=torch.int64, device="cuda")
    word = 32 if max(cx.params.q) < 2**30 else 64
    s = torch.cuda.current_stream()
    for _ in range(3):
        cx.ntt_forward(data, limbs=L, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        cx.ntt_forward(data, limbs=L, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    logn = n.bit_length() - 1
    bfly = polys * L * (n // 2) * logn
    peak = C.c_double()
    nat.call("lb_bench_butterfly_peak", cx.params.q[0], 4, 4000, C.byref(peak))
    achieved = bfly / (ms * 1e-3) / 1e9
    hbm_bytes = polys * L * 16 * n
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6552.6))
    per_limb, src = ncu_traffic(lambda k: k.startswith("ntt_forward_kernel<14, unsigned int, unsigned long>")) \
        if word == 32 else (None, None)  # the generic limb-batch API (u64 limbs)
    return {
        "kernel": f"ntt_forward_kernel<14, u{word}> ({polys * L} limbs of n={n}, "
                  f"{max(cx.params.q).bit_length()}-bit q, {word}-bit words)",
        "bound": "int", "achieved": achieved, "peak": peak.value / 1e9, "unit": "Gbutterfly/s",
        "frac": achieved / (peak.value / 1e9),
        "peak_source": "measured live: register-resident Shoup butterfly microbenchmark (lb_bench_butterfly_peak)",
        "traffic": per_limb * polys * L if per_limb else None,
        "traffic_source": src,
        "launch_ms": ms,
        "limb_transforms_per_s": polys * L / (ms * 1e-3),
        "hbm_view": {"achieved_gbs": hbm_bytes / (ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                     "frac": hbm_bytes / (ms * 1e-3) / 1e9 / hbm_peak, "algorithmic_bytes_per_launch": hbm_bytes},
    }


def ks_roofline(cx, count: int, reps: int = 10) -> dict:
    """The dominant unit: one key switch (inverse NTT of the input, fused
    ModUp+NTT+key MAC over Q∪P, inverse NTT of the P limbs, fused ModDown),
    i.e. ks_inner_kernel + moddown_kernel + ntt_inverse_kernel (~80% of the
    step's device time), timed with CUDA events on its launch stream over a
    batch of `count` ciphertext rotations.

    Algorithmic work = modular (Shoup) products per ciphertext: one per NTT
    butterfly, per ModUp base-conversion term, per key MAC, per ModDown
    conversion term and P^-1 scaling. Peak = the live butterfly
    microbenchmark (one Shoup product + three ALU ops each), so the fraction
    is conservative; the butterfly-only view is reported beside it."""
    import ctypes as C

    import torch

    from paper_1812_10659_b200 import _native as nat
    from paper_1812_10659_b200.bfv import galois_exponent_columns

    n, L, K, dnum = cx.n, cx.L, cx.K, cx.dnum
    alpha = -(-L // dnum)
    digits = [min(L, (j + 1) * alpha) - j * alpha for j in range(dnum)]
    transforms = L + sum(L + K - a for a in digits) + 2 * K + 2 * L
    logn = n.bit_length() - 1
    bfly = transforms * (n // 2) * logn
    modup = sum(a * (L + K - a) for a in digits if a > 1) * n
    mac = 2 * dnum * (L + K) * n
    moddown = ((K * 2 * L) if K > 1 else 0) * n + 2 * L * n
    products = bfly + modup + mac + moddown
    ct = torch.randint(0, min(cx.params.q), (count, 2, L, n), dtype=cx.res_dtype, device="cuda")
    out = torch.empty_like(ct)
    g = galois_exponent_columns(n, 1)
    s = torch.cuda.current_stream()
    for _ in range(3):
        cx.rotate(ct, g, out=out, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        cx.rotate(ct, g, out=out, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    word = 32 if max(cx.params.q) < 2**30 else 64
    peak = C.c_double()
    nat.call("lb_bench_butterfly_peak", cx.params.q[0], 4, 4000, C.byref(peak))
    peak_g = peak.value / 1e9
    achieved = count * products / (ms * 1e-3) / 1e9
    achieved_bfly = count * bfly / (ms * 1e-3) / 1e9
    del ct, out
    # HBM view: the compulsory bytes of one key switch are the input
    # ciphertext read, the output written, and the Galois key (2*dnum*(L+K)
    # limbs) read once per launch set (it is shared by all `count` rotations).
    wb = word // 8
    alg_bytes = count * 4 * L * n * wb + 2 * dnum * (L + K) * n * wb
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6552.6))
    per_ct, src = None, None
    if word == 32:
        try:
            tj = json.loads(TRAFFIC_JSON.read_text())
            if tj["params"]["L"] == L and tj["params"]["K"] == K:
                per_ct = tj["key_switch_bytes_per_ciphertext"]
                src = f"{TRAFFIC_JSON.relative_to(ROOT)}: ks_inner + moddown + the two inverse NTTs, per ciphertext"
        except Exception:
            pass
    return {
        "kernel": f"key switch = ntt_inverse + ks_inner_kernel + ntt_inverse(P) + moddown_kernel, u{word} words, "
                  f"{count} ciphertext rotations per launch set (n={n}, L={L}, K={K}, dnum={dnum})",
        "bound": "int", "achieved": achieved, "peak": peak_g, "unit": "G Shoup products/s",
        "frac": achieved / peak_g,
        "peak_source": "measured live: register-resident Shoup butterfly microbenchmark (lb_bench_butterfly_peak)",
        "traffic": per_ct * count if per_ct else None,
        "traffic_unit": "bytes per launch set (DRAM read + write)",
        "traffic_source": src,
        "algorithmic": f"per ciphertext: {transforms} limb transforms ({bfly} butterflies) + {modup} ModUp + "
                       f"{mac} MAC + {moddown} ModDown products",
        "butterflies_only": {"achieved": achieved_bfly, "frac": achieved_bfly / peak_g},
        "launch_set_ms": ms, "rotations_per_s": count / (ms * 1e-3),
        "hbm_view": {"achieved_gbs": alg_bytes / (ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                     "frac": alg_bytes / (ms * 1e-3) / 1e9 / hbm_peak,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "traffic_over_algorithmic": (per_ct * count / alg_bytes) if per_ct else None},
    }


def run_ours(a, world, rank, local):
    import numpy as np
    import torch

    from paper_1812_10659_b200 import _native as nat
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session, plan_counters
    torch.cuda.set_device(local)
    cfg, strategy, default_batch, net, prm = workload_objects(a.workload, a.word)
    cx = BfvContext(prm)
    B = a.batch or default_batch
    # grow the allocation pool up front (half of the free device memory):
    # mid-run pool growth maps and clears fresh memory, a >1 s stall
    free, _ = torch.cuda.mem_get_info()
    if os.environ.get("LB_POOL_RESERVE", "1") != "0":
        nat.call("lb_pool_reserve", cx.handle, int(free * 0.5))
    sess = Session(cx, net, strategy, B)
    # images of this rank: a disjoint contiguous range of the job's image set
    from paper_1812_10659_b200.shard import shard_range

    imgs = nets.images(cfg, net, B, start=shard_range(world * B, world, rank).start)
    dev_imgs = torch.from_numpy(imgs).cuda()
    counters, _, _ = plan_counters(net, strategy, prm.n)
    rot_per_image = int(counters[:, 5:7].sum()) * len(prm.t)
    s = torch.cuda.current_stream()

    # warm-up: key generation, plaintext encoding, pool growth
    sess.encrypt(dev_imgs, on_device=True)

    def untimed_step() -> float:
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(s)
        sess.execute()
        w1.record(s)
        torch.cuda.synchronize()
        return w0.elapsed_time(w1)

    warm = [untimed_step() for _ in range(a.warmup)]
    # the end-to-end path allocates differently (input encryption, decryption):
    # run it once before any timed region so the stream-ordered pool has grown
    # to the footprint of both paths
    host_imgs = np.ascontiguousarray(imgs)
    scores = np.zeros((B, sess.outputs, 4), dtype=np.uint64)
    sess.run_raw(host_imgs, scores, False, False, want_counters=False, want_times=False)
    sess.encrypt(dev_imgs, on_device=True)
    # settle: a fresh box occasionally shows slow steps right after start-up
    # (pool growth, lazy module loads); keep warming (at most 8 more, untimed)
    # until three consecutive steps agree within 3%
    warm.append(untimed_step())
    for _ in range(8):
        last = warm[-3:]
        if len(last) == 3 and max(last) - min(last) <= 0.03 * min(last):
            break
        warm.append(untimed_step())

    # ---- value: HE steps, encrypted inputs resident in HBM ----
    launches0 = int(nat.lib().lb_launch_count())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(s)
        for i in range(a.steps):
            sess.execute()
            marks[i].record(s)
        e1.record(s)
        torch.cuda.synchronize()
        barrier(world)
    launches = int(nat.lib().lb_launch_count()) - launches0
    step_ms = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i]) for i in range(1, a.steps)]
    elapsed = max_over_ranks(world, e0.elapsed_time(e1) / 1e3)
    value = world * B * a.steps / elapsed

    # ---- e2e: host images -> encrypt -> HE steps -> decrypt -> host scores ----
    # warm until two consecutive end-to-end runs agree within 5% (at most 4):
    # the first runs in a fresh process grow the allocation pool
    e2e_warm = []
    for _ in range(4):
        t0 = time.perf_counter()
        sess.run_raw(host_imgs, scores, False, False, want_counters=False, want_times=False)
        e2e_warm.append(time.perf_counter() - t0)
        if len(e2e_warm) >= 2 and abs(e2e_warm[-1] - e2e_warm[-2]) <= 0.05 * min(e2e_warm[-2:]):
            break
    barrier(world)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(a.steps):
        sess.run_raw(host_imgs, scores, False, False, want_counters=False, want_times=False)
    e1.record(s)
    torch.cuda.synchronize()
    barrier(world)
    e2e_elapsed = max_over_ranks(world, e0.elapsed_time(e1) / 1e3)
    e2e_value = world * B * a.steps / e2e_elapsed

    extras = {}
    if rank == 0 and not a.no_extras:
        del sess
        torch.cuda.empty_cache()
        # single-image latency (server-side HE steps, and end to end)
        one = Session(cx, net, strategy, 1)
        one_img = torch.from_numpy(imgs[:1].copy()).cuda()
        one.encrypt(one_img, on_device=True)
        for _ in range(3):
            one.execute()
        torch.cuda.synchronize()
        lat = []
        for _ in range(5):
            e0.record(s)
            one.execute()
            e1.record(s)
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1))
        sc1 = np.zeros((1, one.outputs, 4), dtype=np.uint64)
        lat_e2e = []
        for _ in range(3):
            t0 = time.perf_counter()
            one.run_raw(np.ascontiguousarray(imgs[:1]), sc1, False, False, want_counters=False, want_times=False)
            lat_e2e.append((time.perf_counter() - t0) * 1e3)
        del one
        torch.cuda.empty_cache()
        extras["latency_ms"] = {"he_steps": min(lat), "e2e": min(lat_e2e), "images": 1}
        # roofline of the dominant unit (the key switch, at a typical plan
        # launch size) and of its NTT component alone
        extras["roofline"] = ks_roofline(cx, 16 * len(prm.t))
        ks_limbs = B * len(prm.t) * prm.dnum * (prm.L + prm.K - 1)
        extras["roofline_ntt"] = ntt_roofline(cx, ks_limbs)
        # CPU baseline: the reference on this host, one thread, bounded sample
        try:
            from oracle import refbind as R

            if R.available() and a.workload == "lola-mnist":
                ips, wall = cpu_reference_throughput(a.cpu_sample, 1)
                extras["cpu_baseline"] = {
                    "value": ips, "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": f"{a.cpu_sample} images, reference packnn ring backend (plaintext semantics, no "
                              f"encryption), encode + HE steps, decode excluded; {wall:.1f} s"}
        except Exception as exc:  # reported, never fatal to the GPU number
            extras["cpu_baseline"] = {"value": None, "error": str(exc)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": elapsed / a.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32" if max(prm.q) < 2**30 else "u64",
            "data": "synthetic (SplitMix64-seeded pixels and weights)",
            "config": {"workload": f"{strategy} cfg{cfg} batched throughput", "images_per_gpu_per_step": B,
                       "n": prm.n, "plain_primes": len(prm.t), "L": prm.L, "K": prm.K, "dnum": prm.dnum,
                       "q_bits": max(prm.q).bit_length(), "residue_storage": "u32 words in HBM when every "
                       "ciphertext and special prime < 2^30, else u64", "parallelism": f"images sharded over {world} GPU(s), no collective",
                       "l2": "working set (encrypted batch, GBs) far larger than the 126 MB L2"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(host_imgs.nbytes) * world,
                    "d2h_bytes_per_step": int(scores.nbytes) * world},
            "gpu_launches": launches,
            "step_ms": [round(v, 3) for v in step_ms],
            "warmup_ms": [round(v, 3) for v in warm],
            "clocks": clk.summary(),
            "rotations_per_s": value * rot_per_image,
            "key_switches_per_image": rot_per_image + int(counters[:, 0].sum()) * len(prm.t),
        }
        line.update(extras)
        print(json.dumps(line))


def main():
    a = parse()
    world, rank, local = dist_setup(a.gpus)
    if a.impl == "reference":
        run_reference(a, world, rank)
    else:
        run_ours(a, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
