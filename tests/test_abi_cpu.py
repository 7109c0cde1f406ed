"""The C-ABI library loads without a GPU and exports every symbol
include/lola_b200.h declares; host-only entry points work on CPU."""
from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1812_10659_b200 import _native as nat
from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.context import find_primes
from paper_1812_10659_b200.lola import plan_counters

HEADER = Path(__file__).resolve().parents[1] / "include" / "lola_b200.h"


def declared() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(lb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = C.CDLL(str(nat.LIB_PATH))
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    bound = set(nat.declared_symbols())
    import paper_1812_10659_b200.evaluator  # registers the Evaluator signatures  # noqa: F401
    import paper_1812_10659_b200.lola  # registers the LoLa signatures  # noqa: F401

    bound |= set(nat.declared_symbols())
    assert set(declared()) <= bound


def test_find_primes_host_only():
    ps = find_primes(60, 16, 4)
    assert len(set(ps)) == 4 and all(p < 2**60 and (p - 1) % 2**16 == 0 for p in ps)
    with pytest.raises(ValueError):
        find_primes(70, 16, 1)


def test_galois_exponents_match_reference():
    from oracle import refbind as R

    for n in (4096, 16384):
        for k in (1, 2, 3, 100, n // 2 - 1):
            assert nat.lib().lb_galois_exponent_columns(n, k) == R.galois_exponent_columns(n, k)
        assert nat.lib().lb_galois_exponent_rows(n) == R.galois_exponent_rows(n)


def test_plan_rejects_bad_networks():
    net = nets.lola_mnist_net()
    with pytest.raises(ValueError):
        plan_counters(net, "no-such-strategy", 16384)
    with pytest.raises(ValueError):
        plan_counters(net, "lola-mnist", 1024)  # 845 combined values do not fit slot row 0


def test_window_matrix_threshold_option():
    """PlanOptions.window_matrix_threshold (plan.hpp:35-41, plan.cpp:375-380):
    lola-cifar's interior window stage (83*6*6 * 163 = 487,092 entries) is
    accepted at the default and rejected once the threshold reaches it."""
    net = nets.lola_cifar_net(config=4)
    vol = 83 * 6 * 6 * 163
    cnt, _, _ = plan_counters(net, "lola-cifar", 16384, window_matrix_threshold=vol - 1)
    assert cnt.shape[0] == 7
    with pytest.raises(ValueError):
        plan_counters(net, "lola-cifar", 16384, window_matrix_threshold=vol)
