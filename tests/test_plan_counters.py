"""CPU: the plan builder's predicted per-step counters equal the reference's
measured counters (slot backend) and its golden traces; no GPU needed."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import refbind as R
from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.lola import plan_counters
from paper_1812_10659_b200.params import REFERENCE_DEFAULT_PRIMES, plain_primes

CASES = [
    ("lola-mnist", nets.lola_mnist_net, 16384, 5, [2, 24, 125, 7, 356, 213, 11]),
    ("lola-mnist", nets.lola_mnist_net, 8192, 5, [2, 36, 125, 13, 411, 268, 11]),
    ("lola-dense-mnist", nets.lola_mnist_net, 16384, 5, [2, 49, 125, 32, 356, 237, 11]),
    ("lola-small", nets.lola_small_net, 8192, 2, [1, 10, 125, 0, 235, 104, 0]),
    ("lola-mnist", nets.toy_net, 4096, 3, None),
    ("cryptonets-simd", nets.toy_net, 4096, 3, None),
]


@pytest.mark.parametrize("strategy,make,n,T,totals", CASES, ids=[f"{c[0]}-{c[2]}-{c[1].__name__}" for c in CASES])
def test_counters_match_reference(strategy, make, n, T, totals):
    net = make()
    mine, depth, _ = plan_counters(net, strategy, n)
    x = nets.images(0, net, 1)[0]
    _, ref, _ = R.run_plan(net, strategy, n, plain_primes(n, T) if T > 3 else REFERENCE_DEFAULT_PRIMES[:T] if n <= 16384 else plain_primes(n, T), x, ring=False)
    assert np.array_equal(mine, ref)
    if totals is not None:
        assert mine.sum(0).tolist() == totals


def test_cifar_counters_match_golden_totals():
    # proj/tests/golden/lola_cifar.txt:10 — the 83/163-map geometry at n=16384
    mine, depth, peak = plan_counters(nets.lola_cifar_net(), "lola-cifar", 16384)
    assert mine.sum(0).tolist() == [2, 8160, 15936, 4075, 81265, 53177, 4075]
    assert depth == 2 and peak == 4075


def test_cryptonets_simd_counters_match_golden():
    # proj/tests/golden/cryptonets_simd.txt:1-10 — the CIFAR net as per-value
    # weighted sums at n=8192, every step
    mine, depth, peak = plan_counters(nets.lola_cifar_net(), "cryptonets-simd", 8192)
    assert mine.tolist() == [[0, 0, 49975296, 0, 49975296, 0, 0], [16268, 0, 0, 0, 0, 0, 0],
                             [0, 0, 66292100, 0, 66292100, 0, 0], [4075, 0, 0, 0, 0, 0, 0],
                             [0, 0, 40750, 0, 40750, 0, 0]]
    assert mine.sum(0).tolist() == [20343, 0, 116308146, 0, 116308146, 0, 0]
    assert depth == 2 and peak == 16268


def test_strategy_mismatch_is_rejected():
    with pytest.raises(ValueError):
        plan_counters(nets.lola_small_net(), "lola-mnist", 8192)
