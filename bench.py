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
    "lola-cifar": (4, "lola-cifar", 2),  # 4,075 live messages x 35 GB per image: B=2 fits 180 GB (B=4 does not)
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


DATA = "synthetic (SplitMix64-seeded pixels and weights)"


def workload_config(a, cfg, strategy, B, prm, world) -> dict:
    """The `config` object of both arms (identical, so the driver compares
    like with like)."""
    return {"workload": f"{strategy} cfg{cfg} batched throughput", "images_per_gpu_per_step": B,
            "n": prm.n, "plain_primes": len(prm.t), "L": prm.L, "K": prm.K, "dnum": prm.dnum,
            "q_bits": max(prm.q).bit_length(), "residue_storage": "u32 words in HBM when every "
            "ciphertext and special prime < 2^30, else u64",
            "parallelism": f"images sharded over {world} GPU(s), no collective",
            "l2": "working set (encrypted batch, GBs) far larger than the 126 MB L2"}


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
    ap.add_argument("--ref-procs", type=int, default=0,
                    help="reference arm: worker processes (default: every host core this process may use)")
    ap.add_argument("--word", type=int, default=32, choices=[32, 64],
                    help="RNS word: 32 = 29/30-bit primes (32-bit word kernels, u32 residues; default), "
                         "64 = 54/60-bit primes")
    return ap.parse_args()


# ---- distributed plumbing -----------------------------------------------------------

def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_if_needed(a) -> None:
    """`--gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N ranks (one per GPU) and exit with its status,
    so a multi-GPU request can never silently measure one GPU. Under torchrun,
    WORLD_SIZE must equal --gpus."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != a.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {a.gpus}")
        return
    if a.gpus <= 1 or a.impl == "reference":
        return  # the reference arm runs on rank 0 only
    import torch

    have = torch.cuda.device_count()
    if have < a.gpus and not SAME_DEVICE:
        raise SystemExit(f"bench.py: --gpus {a.gpus} requested but only {have} CUDA device(s) are visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.stderr.write("bench.py: relaunching under torch.distributed.run: " + " ".join(cmd) + "\n")
    sys.exit(subprocess.call(cmd))


# Functional test hook (tests/test_bench_ranks_gpu.py): LB_RANKS_ON_ONE_GPU=1
# puts every rank on cuda:0 over gloo, to exercise the multi-rank path on a
# one-GPU box. Its timings are meaningless (ranks share the GPU) and it is
# never the driver's configuration.
SAME_DEVICE = os.environ.get("LB_RANKS_ON_ONE_GPU") == "1"
COLL_DEVICE = "cpu" if SAME_DEVICE else "cuda"


def dist_setup(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SAME_DEVICE:
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        if torch.cuda.device_count() <= local:
            raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but {torch.cuda.device_count()} "
                             "device(s) are visible")
        torch.cuda.set_device(local)
        if SAME_DEVICE:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    from paper_1812_10659_b200.shard import barrier as _b

    _b(world)


def max_over_ranks(world, value: float) -> float:
    from paper_1812_10659_b200.shard import max_over_ranks as _m

    return _m(value, world, device=COLL_DEVICE)


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
# The reference arm never loads this repo's device library: parameter sets
# come from params.py (pure Python) and nets.py (numpy); the work runs in
# oracle/_ref/libpackref.so (the unmodified reference compiled in place).

_REF = {}


def _ref_init(workload: str, word: int):
    """Worker start-up (untimed): network, EvalContext and plan built once."""
    from oracle import refbind as R

    cfg, strategy, _, net, prm = workload_objects(workload, word)
    _REF["net"], _REF["cfg"] = net, cfg
    _REF["session"] = R.RefSession(net, strategy, prm.n, prm.t, ring=True, threads=1)


def _ref_image(i: int) -> float:
    """One image of the workload's seeded set: encode + every HE step (the
    per-image work of plan.encode_input + execute); returns its seconds."""
    from paper_1812_10659_b200 import nets

    x = nets.images(_REF["cfg"], _REF["net"], 1, start=i)[0]
    _, t = _REF["session"].run(x)
    return float(t[0] + t[1])


def _ref_ready(_):
    return os.getpid()


class RefPool:
    """`procs` single-thread reference workers, created once (before warm-up)."""

    def __init__(self, workload: str, word: int, procs: int):
        import multiprocessing as mp

        self.procs = procs
        self.pool = mp.get_context("spawn").Pool(procs, initializer=_ref_init, initargs=(workload, word))
        self.pool.map(_ref_ready, range(procs), chunksize=1)

    def run(self, images: range) -> float:
        """Wall seconds for every image of `images`, spread over the workers."""
        t0 = time.perf_counter()
        self.pool.map(_ref_image, list(images), chunksize=max(1, -(-len(images) // self.procs)))
        return time.perf_counter() - t0

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_reference_latency(workload: str, word: int, threads: int, images: int = 2) -> float:
    """The reference's single-image latency with `threads` kernel threads
    (--threads, proj/src/kernels.cpp:161-195: matvec_rowmajor's row fan-out),
    encode + every plan step, best of `images` runs; seconds."""
    from oracle import refbind as R
    from paper_1812_10659_b200 import nets

    cfg, strategy, _, net, prm = workload_objects(workload, word)
    rs = R.RefSession(net, strategy, prm.n, prm.t, ring=True, threads=threads)
    x = nets.images(cfg, net, 1)[0]
    best = float("inf")
    for _ in range(images):
        _, t = rs.run(x)
        best = min(best, float(t[0] + t[1]))
    return best


def cpu_reference_single(workload: str, word: int, images: int) -> tuple[float, float]:
    """One thread, this process: (images/s, seconds) over `images` images."""
    _ref_init(workload, word)
    _ref_image(0)  # warm (page-in, first allocations)
    t = sum(_ref_image(i) for i in range(images))
    return images / t, t


# ---- reference arm ----------------------------------------------------------------------

def run_reference(a, world, rank):
    if rank != 0:
        return
    from oracle import refbind as R

    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libpackref.so not built"}))
        return
    cfg, strategy, default_batch, net, prm = workload_objects(a.workload, a.word)
    B = a.batch or default_batch
    procs = min(a.ref_procs or host_cores(), B)
    pool = RefPool(a.workload, a.word, procs)
    images = range(0, B)  # rank 0's image range of our arm
    for _ in range(a.warmup):
        pool.run(images)
    per_step = [pool.run(images) for _ in range(a.steps)]
    pool.close()
    wall = sum(per_step)
    value = a.steps * B / wall
    sample = (f"{B} images per step (the same seeded images as our arm's rank 0), {procs} single-thread worker "
              f"processes created once before warm-up, each with its network, EvalContext and plan built once; "
              f"per image: plan.encode_input + every plan step on the reference ring backend (plaintext "
              f"semantics, no encryption); decode excluded (the Boost stand-in BigInt is not representative)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": wall / a.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": DATA,
        "config": workload_config(a, cfg, strategy, B, prm, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms": [round(v * 1e3, 1) for v in per_step],
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


def _peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def butterfly_peak(q: int) -> float:
    """Live integer roof of the word size of prime q: sustained
    register-resident Harvey/Shoup butterflies per second (G/s)."""
    import ctypes as C

    from paper_1812_10659_b200 import _native as nat

    peak = C.c_double()
    nat.call("lb_bench_butterfly_peak", q, 4, 4000, C.byref(peak))
    return peak.value / 1e9


_PIPES = {}


def pipe_check() -> dict:
    """Cross-check of the butterfly roof against the FMA-pipe limit: measured
    IMAD and IMAD.HI issue rates (lb_bench_int_pipes); a 32-bit Shoup
    butterfly needs one IMAD.HI and two IMADs on that pipe."""
    import ctypes as C

    from paper_1812_10659_b200 import _native as nat

    if not _PIPES:
        ops = (C.c_double * 5)()
        nat.call("lb_bench_int_pipes", 20000, ops)
        imad, imad_hi = ops[0] / 1e9, ops[1] / 1e9
        bound = 1.0 / (1.0 / imad_hi + 2.0 / imad)
        _PIPES.update({"imad_gops": imad, "imad_hi_gops": imad_hi, "imad_wide_gops": ops[4] / 1e9,
                       "fma_pipe_bound_gbfly_s_u32": bound})
    return dict(_PIPES)


def ntt_roofline(cx, limbs: int, reps: int = 20) -> dict:
    """The hot path's NTT alone: the u32-storage forward and inverse limb
    transforms (ntt_forward_kernel / ntt_inverse_kernel<LOGN, u32, u32>, the
    kernels the key switch launches) over the key switch's limb count at the
    bench batch, timed with CUDA events on their launch stream, against the
    live butterfly peak of the same word size. 64-bit contexts time the u64
    kernels."""
    import torch

    n, L = cx.n, cx.L
    polys = max(1, limbs // L)
    word = 32 if max(cx.params.q) < 2**30 else 64
    dt = torch.int32 if word == 32 else torch.int64
    data = torch.randint(0, min(cx.params.q), (polys, L, n), dtype=dt, device="cuda")
    s = torch.cuda.current_stream()
    res = {}
    for name, fn in (("forward", cx.ntt_forward), ("inverse", cx.ntt_inverse)):
        for _ in range(3):
            fn(data, limbs=L, stream=s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            fn(data, limbs=L, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps
    del data
    logn = n.bit_length() - 1
    bfly = polys * L * (n // 2) * logn
    peak = butterfly_peak(cx.params.q[0])
    ms = (res["forward"] + res["inverse"]) / 2
    achieved = bfly / (ms * 1e-3) / 1e9
    wb = word // 8
    hbm_bytes = polys * L * 2 * wb * n
    hbm_peak = float(_peaks().get("hbm_gbs", 6552.6))
    per_limb, src = (None, None)
    if word == 32:
        f_b, f_s = ncu_traffic(lambda k: k.startswith("ntt_forward_kernel<14, unsigned int, unsigned int"))
        i_b, i_s = ncu_traffic(lambda k: k.startswith("ntt_inverse_kernel<14, unsigned int, unsigned int"))
        if f_b and i_b:
            per_limb, src = (f_b + i_b) / 2, f"{f_s}; {i_s}"
    return {
        "kernel": f"ntt_forward_kernel + ntt_inverse_kernel<{logn}, u{word}, u{word}> (mean; {polys * L} limbs of "
                  f"n={n}, {max(cx.params.q).bit_length()}-bit q, {word}-bit words, u{word} storage)",
        "bound": "int", "achieved": achieved, "peak": peak, "unit": "Gbutterfly/s",
        "frac": achieved / peak,
        "peak_source": "measured live: register-resident Shoup butterfly microbenchmark (lb_bench_butterfly_peak)",
        "traffic": per_limb * polys * L if per_limb else None,
        "traffic_source": src,
        "launch_ms": ms, "forward_ms": res["forward"], "inverse_ms": res["inverse"],
        "frac_forward": bfly / (res["forward"] * 1e-3) / 1e9 / peak,
        "frac_inverse": bfly / (res["inverse"] * 1e-3) / 1e9 / peak,
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

    Algorithmic work = modular (Shoup) products per ciphertext by SURVEY
    §8(d)'s formula: one per NTT butterfly, per ModUp and ModDown
    base-conversion term and per key MAC. Peak = the live butterfly
    microbenchmark (one Shoup product + three ALU ops each), so the fraction
    is conservative; the butterfly-only view is reported beside it."""
    import torch

    from paper_1812_10659_b200.bfv import galois_exponent_columns

    n, L, K, dnum = cx.n, cx.L, cx.K, cx.dnum
    alpha = -(-L // dnum)
    # T = L + dnum (L + K - alpha) + 2K + 2L limb transforms;
    # dnum alpha (L + K - alpha) N ModUp + 2 K L N ModDown conversion MACs;
    # 2 dnum (L + K) N key inner-product MACs
    transforms = L + dnum * (L + K - alpha) + 2 * K + 2 * L
    logn = n.bit_length() - 1
    bfly = transforms * (n // 2) * logn
    modup = dnum * alpha * (L + K - alpha) * n
    mac = 2 * dnum * (L + K) * n
    moddown = 2 * K * L * n
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
    peak_g = butterfly_peak(cx.params.q[0])
    achieved = count * products / (ms * 1e-3) / 1e9
    achieved_bfly = count * bfly / (ms * 1e-3) / 1e9
    del ct, out
    # HBM view: the compulsory bytes of one key switch are the input
    # ciphertext read, the output written, and the Galois key (2*dnum*(L+K)
    # limbs) read once per launch set (it is shared by all `count` rotations).
    wb = word // 8
    alg_bytes = count * 4 * L * n * wb + 2 * dnum * (L + K) * n * wb
    hbm_peak = float(_peaks().get("hbm_gbs", 6552.6))
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
        "peak_cross_check": pipe_check() if word == 32 else None,
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


def parity_check(net, imgs, scores, limit: int = 256) -> dict:
    """Decrypted logits of the timed batch vs forward_integer, the
    reference's integer oracle (proj/src/layers.cpp:560-594), run from
    oracle/_ref as the checker (outside every timed region). Every image when
    the batch has <= `limit`, else an even sample of `limit`."""
    from oracle import refbind as R
    from paper_1812_10659_b200.lola import words_to_int

    B = scores.shape[0]
    idx = list(range(B)) if B <= limit else list(range(0, B, B // limit))[:limit]
    bad = []
    for i in idx:
        got = [words_to_int(scores[i, j]) for j in range(scores.shape[1])]
        if got != R.forward_integer(net, imgs[i]):
            bad.append(i)
    return {"images": len(idx), "mismatches": len(bad), "first_bad": bad[:8],
            "checker": "oracle/_ref forward_integer (proj/src/layers.cpp:560-594)"}


def timed_steps(sess, steps: int) -> float:
    """Device seconds of `steps` HE steps of a session (CUDA events)."""
    import torch

    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        sess.execute()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def value_w64(a, net, strategy, B, imgs) -> dict:
    """The same plan on the 60-bit parameter set (64-bit Shoup words, u64
    residues): device-timed HE steps and the decrypted logits' parity."""
    import numpy as np
    import torch

    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session
    from paper_1812_10659_b200.params import lola_mnist_params

    prm = lola_mnist_params()
    cx = BfvContext(prm)
    sess = Session(cx, net, strategy, B)
    sess.encrypt(torch.from_numpy(imgs).cuda(), on_device=True)
    for _ in range(2):
        sess.execute()
    steps = max(2, min(a.steps, 5))
    sec = timed_steps(sess, steps)
    scores = np.zeros((B, sess.outputs, 4), dtype=np.uint64)
    sess.run_raw(np.ascontiguousarray(imgs), scores, False, False, want_counters=False, want_times=False)
    par = parity_check(net, imgs, scores)
    del sess
    torch.cuda.empty_cache()
    ks = ks_roofline(cx, B * len(prm.t))
    ntt = ntt_roofline(cx, B * len(prm.t) * prm.dnum * (prm.L + prm.K - 1))
    del cx
    torch.cuda.empty_cache()
    return {"value": B * steps / sec, "unit": UNIT, "ms_per_step": sec / steps * 1e3, "steps": steps,
            "images_per_step": B, "dtype": "u64", "q_bits": max(prm.q).bit_length(), "L": prm.L, "K": prm.K,
            "dnum": prm.dnum, "parity": par,
            "roofline": {k: ks[k] for k in ("kernel", "bound", "achieved", "peak", "unit", "frac", "launch_set_ms",
                                             "algorithmic")},
            "roofline_ntt": {k: ntt[k] for k in ("kernel", "bound", "achieved", "peak", "unit", "frac",
                                                 "frac_forward", "frac_inverse", "hbm_view")}}


# BASELINE config 1 grid of the bench's primitive leg: (n, L, K, dnum, bits)
PRIMITIVE_GRID = [(4096, 4, 1, 0, 60), (8192, 6, 2, 3, 60), (16384, 8, 2, 4, 60), (32768, 12, 2, 6, 60),
                  (16384, 10, 5, 2, 29)]


def primitives(batch: int = 64, reps: int = 10) -> list[dict]:
    """Config 1: batches of 64 ciphertexts, NTT limb transforms/s (vs the
    live butterfly roof), ct x pt, ct + ct, rotations and square+relin per
    second, device-timed; with the reference's per-limb CPU times beside."""
    import torch

    from oracle import refbind as R
    from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns
    from paper_1812_10659_b200.params import make_params

    def timed(fn, r):
        for _ in range(2):
            fn()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(r):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / r * 1e-3

    out = []
    for n, L, K, dnum, bits in PRIMITIVE_GRID:
        prm = make_params(n, L=L, T=1, K=K, dnum=dnum, bits=bits, seed=1)
        cx = BfvContext(prm)
        peak = butterfly_peak(prm.q[0])
        vals = torch.randint(-1000, 1000, (batch, n), dtype=torch.int64, device="cuda")
        ct = cx.encrypt_slots(vals, id_base=1)
        ct2 = cx.encrypt_slots(vals, id_base=batch + 1)
        pm, _ = cx.encode_plain(vals[0], add=False)
        o = torch.empty_like(ct)
        limbs = torch.randint(0, min(prm.q), (batch * 2, L, n), dtype=cx.res_dtype, device="cuda")
        g = galois_exponent_columns(n, 1)
        cx.keygen(g)
        cx.keygen(0)
        t_fwd = timed(lambda: cx.ntt_forward(limbs, limbs=L), reps)
        t_inv = timed(lambda: cx.ntt_inverse(limbs, limbs=L), reps)
        t_mp = timed(lambda: cx.mul_plain(ct, pm, out=o), reps)
        t_add = timed(lambda: cx.add(ct, ct2, out=o), reps)
        t_rot = timed(lambda: cx.rotate(ct, g, out=o), max(2, reps // 2))
        t_sq = timed(lambda: cx.mul(ct, ct, out=o), max(2, reps // 2))
        nl = batch * 2 * L
        bfly = nl * (n // 2) * (n.bit_length() - 1)
        cpu = R.time_primitives(prm.q[0], n, 3)
        out.append({
            "n": n, "L": L, "K": K, "dnum": prm.dnum, "q_bits": bits, "batch": batch,
            "word": "u32" if cx.res_dtype == torch.int32 else "u64",
            "ntt_fwd_limbs_per_s": nl / t_fwd, "ntt_inv_limbs_per_s": nl / t_inv,
            "ntt_fwd_frac": bfly / t_fwd / 1e9 / peak, "ntt_inv_frac": bfly / t_inv / 1e9 / peak,
            "butterfly_peak_gbfly_s": peak,
            "ct_pt_per_s": batch / t_mp, "ct_add_per_s": batch / t_add, "rotations_per_s": batch / t_rot,
            "square_relin_per_s": batch / t_sq,
            "cpu_reference_per_limb_s": cpu,
        })
        del cx, ct, ct2, o, limbs, pm, vals
        torch.cuda.empty_cache()
    return out


def cpu_bfv_baseline(prm, ks_per_image: int) -> dict:
    """Our CPU BFV oracle (oracle/bfv_oracle.cpp, one thread) running the
    plan's key-switch mix: seconds per rotation (automorphism + hybrid key
    switch, key made once) x key switches per image."""
    import numpy as np

    from oracle.bfvbind import Oracle

    o = Oracle.from_params(prm)
    rng = np.random.default_rng(0)
    ct = np.stack([np.stack([rng.integers(0, q, prm.n, dtype=np.uint64) for q in prm.q]) for _ in range(2)])
    _, sec = o.time_rotate(ct, 3, 2)
    per = sec / 2
    return {"value": 1.0 / (per * ks_per_image), "unit": UNIT, "cores": 1, "kind": "port",
            "seconds_per_key_switch": per, "key_switches_per_image": ks_per_image,
            "sample": f"2 rotations (n={prm.n}, L={prm.L}, K={prm.K}, dnum={prm.dnum}) on the CPU BFV oracle, "
                      f"one thread; inferences/s = 1 / (seconds per key switch x {ks_per_image} key switches per "
                      "image), key switching only (a lower bound on a CPU BFV inference's time)"}


def run_ours(a, world, rank, local):
    import numpy as np
    import torch

    from paper_1812_10659_b200 import _native as nat
    from paper_1812_10659_b200 import nets
    from paper_1812_10659_b200.bfv import BfvContext
    from paper_1812_10659_b200.lola import Session, plan_counters
    from paper_1812_10659_b200.shard import shard_range, sum_over_ranks
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
    imgs = nets.images(cfg, net, B, start=shard_range(world * B, world, rank).start)
    dev_imgs = torch.from_numpy(imgs).cuda()
    counters, _, _ = plan_counters(net, strategy, prm.n)
    rot_per_image = int(counters[:, 5:7].sum()) * len(prm.t)
    ks_per_image = rot_per_image + int(counters[:, 0].sum()) * len(prm.t)
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
    scores[:] = 0
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

    # ---- parity of exactly what was timed: the last e2e step's decrypted
    # logits of every image of this rank vs the reference's integer oracle ----
    par = parity_check(net, imgs, scores)
    mism = int(sum_over_ranks(float(par["mismatches"]), world, device=COLL_DEVICE))
    checked = int(sum_over_ranks(float(par["images"]), world, device=COLL_DEVICE))
    parity = {"images": checked, "mismatches": mism, "checker": par["checker"],
              "of": f"decrypted logits of the last timed e2e step, {'all' if checked == world * B else 'a sample of'} "
                    f"{world * B} images"}
    if rank == 0 and par["first_bad"]:
        parity["first_bad_rank0"] = par["first_bad"]

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
        lat_e2e = []  # (no graph)
        for _ in range(3):
            t0 = time.perf_counter()
            one.run_raw(np.ascontiguousarray(imgs[:1]), sc1, False, False, want_counters=False, want_times=False)
            lat_e2e.append((time.perf_counter() - t0) * 1e3)
        # the same with the plan replayed as one CUDA graph
        one.set_graph(True)
        one.encrypt(one_img, on_device=True)
        for _ in range(3):
            one.execute()
        torch.cuda.synchronize()
        lat_g = []
        for _ in range(5):
            e0.record(s)
            one.execute()
            e1.record(s)
            torch.cuda.synchronize()
            lat_g.append(e0.elapsed_time(e1))
        lat_ge = []
        for _ in range(3):
            t0 = time.perf_counter()
            one.run_raw(np.ascontiguousarray(imgs[:1]), sc1, False, False, want_counters=False, want_times=False)
            lat_ge.append((time.perf_counter() - t0) * 1e3)
        g_par = parity_check(net, imgs[:1], sc1)
        extras["latency_ms"] = {"he_steps": min(lat_g), "e2e": min(lat_ge), "images": 1, "cuda_graph": True,
                                "he_steps_no_graph": min(lat), "e2e_no_graph": min(lat_e2e),
                                "graph_parity": g_par["mismatches"] == 0}
        del one
        torch.cuda.empty_cache()
        # roofline of the dominant unit (the key switch, at the size the plan
        # launches it: every rotation of the step runs over all B x T
        # ciphertexts of the batch) and of its NTT component alone
        extras["roofline"] = ks_roofline(cx, B * len(prm.t))
        ks_limbs = B * len(prm.t) * prm.dnum * (prm.L + prm.K - 1)
        extras["roofline_ntt"] = ntt_roofline(cx, ks_limbs)
        if a.workload == "lola-mnist" and a.word == 32:
            del cx
            torch.cuda.empty_cache()
            extras["value_w64"] = value_w64(a, net, strategy, B, imgs)
            extras["primitives"] = primitives()
        # CPU baselines on this host: the reference (one thread, bounded
        # sample) and our CPU BFV oracle's key switching
        try:
            from oracle import refbind as R

            if R.available():
                ips, sec = cpu_reference_single(a.workload, a.word, a.cpu_sample)
                extras["cpu_baseline"] = {
                    "value": ips, "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": f"{a.cpu_sample} images of the workload, reference packnn ring backend (plaintext "
                              f"semantics, no encryption), network/EvalContext/plan built once, per image "
                              f"encode + every plan step, decode excluded; {sec:.1f} s"}
            extras["cpu_baseline_bfv"] = cpu_bfv_baseline(prm, ks_per_image)
            if R.available():
                cores = host_cores()
                extras["cpu_latency_ms"] = {
                    "threads_1": cpu_reference_latency(a.workload, a.word, 1) * 1e3,
                    f"threads_{cores}": cpu_reference_latency(a.workload, a.word, cores) * 1e3,
                    "what": "reference ring backend, one image, encode + every plan step, --threads 1 and "
                            "--threads $(nproc) (kernels.cpp:161-195 fans matvec_rowmajor rows out)"}
        except Exception as exc:  # reported, never fatal to the GPU number
            extras.setdefault("cpu_baseline", {"value": None, "error": str(exc)[:200]})

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": elapsed / a.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32" if max(prm.q) < 2**30 else "u64",
            "data": DATA,
            "config": workload_config(a, cfg, strategy, B, prm, world),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(host_imgs.nbytes) * world,
                    "d2h_bytes_per_step": int(scores.nbytes) * world},
            "parity": parity,
            "gpu_launches": launches,
            "step_ms": [round(v, 3) for v in step_ms],
            "warmup_ms": [round(v, 3) for v in warm],
            "clocks": clk.summary(),
            "rotations_per_s": value * rot_per_image,
            "key_switches_per_image": ks_per_image,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    if mism:
        sys.stderr.write(f"bench.py: PARITY FAILURE: {mism} of {checked} images' decrypted logits differ from "
                         "forward_integer\n")
        sys.exit(3)


def main():
    a = parse()
    relaunch_if_needed(a)
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
