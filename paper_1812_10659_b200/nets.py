"""Integer network descriptions and the seeded synthetic BASELINE configs.

A `Network` mirrors the reference's quantized network
(proj/include/packnn/layers.hpp:100-123): linear stages (window stencil or
matrix) with a squaring after every stage but the last. MNIST / CIFAR-10 and
trained weights are not in this image; SplitMix64-seeded uniform integers with
the BASELINE.json shapes and ranges stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """count outputs of SplitMix64 started at `seed` (portable, numpy-vectorized)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & (2**64 - 1)) + _GAMMA * (np.arange(1, count + 1, dtype=np.uint64))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_ints(seed: int, count: int, lo: int, hi: int) -> np.ndarray:
    """value = lo + r mod (hi - lo + 1) for SplitMix64 outputs r."""
    r = splitmix64(seed, count)
    return (lo + (r % np.uint64(hi - lo + 1)).astype(np.int64)).astype(np.int64)


def seed_of(config: int, tensor: int, index: int = 0) -> int:
    """Seeds are (config, tensor-id, image-index)."""
    return (config << 48) ^ (tensor << 32) ^ index


@dataclass
class Stage:
    is_conv: bool
    rows: int                      # conv: maps; dense: outputs
    cols: int                      # conv: window volume; dense: inputs
    weights: np.ndarray            # rows x cols int64
    bias: np.ndarray | None = None
    win: tuple = (1, 1)
    stride: tuple = (1, 1)
    pad: tuple = (0, 0, 0, 0)      # top, left, bottom, right


@dataclass
class Network:
    input_shape: tuple             # (channels, h, w)
    stages: list = field(default_factory=list)
    input_bound: int = 255

    @property
    def input_values(self) -> int:
        c, h, w = self.input_shape
        return c * h * w


def conv_out(h: int, w: int, st: Stage) -> tuple:
    t, l, b, r = st.pad
    return (h + t + b - st.win[0]) // st.stride[0] + 1, (w + l + r - st.win[1]) // st.stride[1] + 1


# ---- BASELINE.json configs ------------------------------------------------------

def lola_mnist_net(config: int = 0, wmax: int = 64) -> Network:
    """Config 0/2: 28x28 -> conv 5 maps 5x5 stride 2 (pads top/left 1, 13x13
    grid as proj/tests/net_builders.hpp:44-46) -> square -> dense 845->100 ->
    square -> dense 100->10. Weights U[-64, 64], zero biases."""
    conv = Stage(True, 5, 25, uniform_ints(seed_of(config, 1), 5 * 25, -wmax, wmax).reshape(5, 25),
                 np.zeros(5, np.int64), win=(5, 5), stride=(2, 2), pad=(1, 1, 0, 0))
    d1 = Stage(False, 100, 845, uniform_ints(seed_of(config, 2), 100 * 845, -wmax, wmax).reshape(100, 845),
               np.zeros(100, np.int64))
    d2 = Stage(False, 10, 100, uniform_ints(seed_of(config, 3), 10 * 100, -wmax, wmax).reshape(10, 100),
               np.zeros(10, np.int64))
    return Network((1, 28, 28), [conv, d1, d2], 255)


def lola_small_net(config: int = 3, wmax: int = 64) -> Network:
    """Config 3: the LoLa-MNIST window stage then dense 845->10."""
    conv = Stage(True, 5, 25, uniform_ints(seed_of(config, 1), 5 * 25, -wmax, wmax).reshape(5, 25),
                 np.zeros(5, np.int64), win=(5, 5), stride=(2, 2), pad=(1, 1, 0, 0))
    d1 = Stage(False, 10, 845, uniform_ints(seed_of(config, 2), 10 * 845, -wmax, wmax).reshape(10, 845),
               np.zeros(10, np.int64))
    return Network((1, 28, 28), [conv, d1], 255)


def lola_cifar_net(config: int = 4, wmax: int = 32) -> Network:
    """Config 4: 3x32x32 -> conv 83 maps 8x8 s2 pad 1 (14x14, 16268 values)
    -> square -> conv 163 maps 6x6 s2 (5x5, 4075) -> square -> dense 10."""
    c1 = Stage(True, 83, 192, uniform_ints(seed_of(config, 1), 83 * 192, -wmax, wmax).reshape(83, 192),
               np.zeros(83, np.int64), win=(8, 8), stride=(2, 2), pad=(1, 1, 1, 1))
    c2 = Stage(True, 163, 83 * 36, uniform_ints(seed_of(config, 2), 163 * 83 * 36, -wmax, wmax).reshape(163, -1),
               np.zeros(163, np.int64), win=(6, 6), stride=(2, 2))
    d = Stage(False, 10, 4075, uniform_ints(seed_of(config, 3), 10 * 4075, -wmax, wmax).reshape(10, 4075),
              np.zeros(10, np.int64))
    return Network((3, 32, 32), [c1, c2, d], 255)


def toy_net(config: int = 9, side: int = 8, maps: int = 2, r1: int = 6, r2: int = 3) -> Network:
    """Small window-front net (shape of proj/tests/net_builders.hpp:89-97):
    side x side input, 3x3 stride-2 window, `maps` maps, r1 and r2 wide
    matrices, small weights and nonzero biases."""
    out = (side - 3) // 2 + 1
    comb = maps * out * out
    conv = Stage(True, maps, 9, uniform_ints(seed_of(config, 1), maps * 9, -2, 2).reshape(maps, 9),
                 uniform_ints(seed_of(config, 4), maps, -3, 3), win=(3, 3), stride=(2, 2))
    d1 = Stage(False, r1, comb, uniform_ints(seed_of(config, 2), r1 * comb, -2, 2).reshape(r1, comb),
               uniform_ints(seed_of(config, 5), r1, -3, 3))
    d2 = Stage(False, r2, r1, uniform_ints(seed_of(config, 3), r2 * r1, -2, 2).reshape(r2, r1),
               uniform_ints(seed_of(config, 6), r2, -3, 3))
    return Network((1, side, side), [conv, d1, d2], 8)


def images(config: int, net: Network, count: int, start: int = 0, lo: int = 0, hi: int = 255) -> np.ndarray:
    """Seeded synthetic inputs [count][input_values] (pixels U{lo..hi})."""
    hi = min(hi, net.input_bound)
    return np.stack([uniform_ints(seed_of(config, 0, start + i), net.input_values, lo, hi) for i in range(count)])
