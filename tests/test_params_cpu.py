"""Shipped BFV parameter sets (paper_1812_10659_b200/params.py): 128-bit
security bound on log2(QP) (HE standard, ternary secret), word-size and
digit-structure invariants the kernels rely on. Host-only (prime search via
the C-ABI, no GPU)."""
import math

import pytest

from paper_1812_10659_b200 import params as P

# HomomorphicEncryption.org standard, 128-bit classical security, ternary secret
MAX_LOG_QP = {4096: 109, 8192: 218, 16384: 438, 32768: 881}

SETS = {
    "lola_mnist_params": P.lola_mnist_params,
    "lola_mnist_params_w32": P.lola_mnist_params_w32,
    "lola_small_params": P.lola_small_params,
    "lola_small_params_w32": P.lola_small_params_w32,
    "lola_cifar_params": P.lola_cifar_params,
    "lola_cifar_params_w32": P.lola_cifar_params_w32,
}


@pytest.mark.parametrize("name", sorted(SETS))
def test_security_bound(name):
    prm = SETS[name]()
    assert prm.log_qp() <= MAX_LOG_QP[prm.n], f"{name}: log2 QP {prm.log_qp():.1f} > {MAX_LOG_QP[prm.n]}"


@pytest.mark.parametrize("name", sorted(SETS))
def test_prime_chain_invariants(name):
    prm = SETS[name]()
    allp = [*prm.q, *prm.p, *prm.b]
    assert len(set(allp)) == len(allp), "ciphertext, special and auxiliary primes must be distinct"
    assert all((v - 1) % (2 * prm.n) == 0 for v in allp), "NTT-friendly: p == 1 mod 2n"
    assert all((t - 1) % (2 * prm.n) == 0 for t in prm.t), "batching: t == 1 mod 2n"
    # the fused key switch feeds unreduced base-conversion sums (< 4 r) into the
    # lazy transform: every Q/P prime within a factor 4 of every other
    qp = [*prm.q, *prm.p]
    assert max(qp) < 4 * min(qp)
    # one word size per context: all below 2^30 (32-bit word kernels) or all 64-bit words
    assert all(v < 2**30 for v in qp) or all(v >= 2**30 for v in qp)
    # digits: dnum digits of alpha = ceil(L / dnum) primes
    assert 1 <= prm.dnum <= prm.L
    # the auxiliary base holds round(t D / Q) for the exact tensor product
    log_b = sum(math.log2(v) for v in prm.b)
    log_q = sum(math.log2(v) for v in prm.q)
    assert log_b >= log_q + math.log2(max(prm.t)) + math.log2(prm.n) + 2


def test_python_prime_search_matches_the_library():
    """params.find_primes (pure Python, used by the parameter sets and the
    reference arm) == lb_find_primes (csrc/host_math.hpp)."""
    from paper_1812_10659_b200 import context, params

    for bits, log_mod, count in ((29, 16, 24), (30, 16, 20), (54, 16, 8), (60, 16, 16), (31, 15, 6)):
        assert params.find_primes(bits, log_mod, count) == context.find_primes(bits, log_mod, count)
    ex = params.find_primes(60, 16, 3)
    assert params.find_primes(60, 16, 3, exclude=ex[:2]) == context.find_primes(60, 16, 3, exclude=ex[:2])
    from oracle import refbind as R

    assert all(R.is_prime(v) for v in params.find_primes(60, 16, 4))


def test_default_seeds_are_fresh():
    from paper_1812_10659_b200 import params

    seeds = {params.lola_mnist_params_w32().seed for _ in range(4)}
    assert len(seeds) == 4 and all(s % 2 == 1 and s < 2**63 for s in seeds)
    assert params.make_params(4096, L=2, seed=5).seed == 5
