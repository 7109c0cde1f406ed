"""BFV-RNS parameter sets for the LoLa configurations (BASELINE.json).

The reference has no ciphertext modulus at all; its only moduli
are the plaintext primes (proj/src/plan.cpp:574 default, and the suggestion
list proj/src/layers.cpp:288-290). Those become our plaintext CRT primes t_j,
each an independent BFV instance. The ciphertext chain Q, the
special primes P (hybrid key switching) and the auxiliary base B (exact
HPS-style multiplication) are chosen here, deterministically.
"""
from __future__ import annotations

from dataclasses import dataclass, field

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime_u64(v: int) -> bool:
    """Deterministic Miller-Rabin for every u64 (the bases of
    proj/src/modular.cpp:22-42; same routine as csrc/host_math.hpp)."""
    if v < 2:
        return False
    for s in _MR_BASES:
        if v % s == 0:
            return v == s
    d, r = v - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_BASES:
        x = pow(a, d, v)
        if x in (1, v - 1):
            continue
        for _ in range(r - 1):
            x = x * x % v
            if x == v - 1:
                break
        else:
            return False
    return True


def find_primes(bits: int, log_mod: int, count: int, exclude=()) -> list[int]:
    """The `count` largest primes below 2^bits that are == 1 mod 2^log_mod,
    skipping `exclude`: the same search as lb_find_primes
    (csrc/host_math.hpp), in pure Python so that parameter sets (and the CPU
    reference arm of bench.py, which must not load the device library) need
    no native code."""
    if bits < log_mod + 2 or bits > 62:
        raise ValueError("bad prime size")
    step = 1 << log_mod
    c = ((1 << bits) - 1) // step * step + 1
    if c >= 1 << bits:
        c -= step
    ex = set(int(e) for e in exclude)
    out: list[int] = []
    while c > step and len(out) < count:
        if c not in ex and is_prime_u64(c):
            out.append(c)
        c -= step
    if len(out) < count:
        raise ValueError("not enough primes of that shape")
    return out

# proj/src/layers.cpp:288-290 — primes == 1 mod 32768, largest first.
SUGGESTED_PLAIN_PRIMES = [2281701377, 2149810177, 2148794369, 2148728833, 2013265921, 1004535809, 998244353]
# proj/src/plan.cpp:574
REFERENCE_DEFAULT_PRIMES = [2148728833, 2148794369, 2149810177]


@dataclass
class BfvParams:
    n: int
    q: list[int]
    p: list[int]
    b: list[int]
    t: list[int]
    dnum: int = 0
    seed: int = 0
    notes: dict = field(default_factory=dict)

    @property
    def L(self) -> int:
        return len(self.q)

    @property
    def K(self) -> int:
        return len(self.p)

    def log_qp(self) -> float:
        import math

        return sum(math.log2(v) for v in (*self.q, *self.p))


def plain_primes(n: int, count: int) -> list[int]:
    """`count` plaintext primes that support degree n: the reference's
    suggestion list first (all == 1 mod 2^15, valid up to n = 16384), then a
    deterministic search for 31-bit primes == 1 mod 2n."""
    ok = [t for t in SUGGESTED_PLAIN_PRIMES if (t - 1) % (2 * n) == 0]
    if len(ok) >= count:
        return ok[:count]
    extra = find_primes(31, (2 * n).bit_length() - 1, count - len(ok), exclude=ok)
    return ok + extra


def make_params(n: int, L: int, T: int = 1, K: int = 1, dnum: int = 0, bits: int = 60, seed: int | None = None,
                plain: list[int] | None = None) -> BfvParams:
    """Ciphertext primes: the L largest `bits`-bit primes == 1 mod 2^16 (so
    one chain serves every n <= 32768); special primes and the auxiliary
    base B are the next ones down, all distinct. B must hold round(t D / Q)
    for the tensor D (|D| < n Q^2 / 4): log2 B >= log2 Q + log2 t + log2 n + 2,
    i.e. L + 1 primes of 60 bits or L + 2 of 30 bits."""
    import math

    log_mod = 16
    extra = max(1, math.ceil((32 + math.log2(n) + 3) / (bits - 1)))
    allp = find_primes(bits, log_mod, L + K + L + extra)
    q, p, b = allp[:L], allp[L:L + K], allp[L + K:]
    t = plain if plain is not None else plain_primes(n, T)
    return BfvParams(n=n, q=q, p=p, b=b, t=t, dnum=dnum or L, seed=fresh_seed() if seed is None else seed)


def fresh_seed() -> int:
    """Key/randomness seed from OS entropy: the default, so two contexts
    never share a secret key. Explicit seeds are for parity tests (the CPU
    oracle reproduces a context from its seed)."""
    import secrets

    return secrets.randbits(63) | 1


# BASELINE.json configs --------------------------------------------------------

def lola_mnist_params(seed: int | None = None) -> BfvParams:
    """Config 0/2: n = 16384, 5 plaintext primes (the runtime
    magnitude bound needs 5), L = 5 ciphertext primes of 60 bits, K = 2
    special primes, dnum = 3 digits of <= 2 primes: log2(QP) = 420 <= 438,
    the HE-standard 128-bit bound for n = 16384 with a ternary secret.
    Measured end-of-network noise ~229 bits against log2(Q / 2t) ~ 268; 35
    limb transforms per key switch (vs 42 with K = 1, dnum = 5), measured
    84 vs 76 images/s on B200."""
    return make_params(16384, L=5, T=5, K=2, dnum=3, seed=seed)


def lola_mnist_params_w32(seed: int | None = None) -> BfvParams:
    """Config 0/2 on 29-bit primes (below 2^30, so every transform and key
    switch runs on 32-bit words): L = 10 ciphertext primes (Q ~ 290 bits),
    K = 5 special primes, dnum = 2 digits of 5 primes (P ~ D_j, so key
    switching adds no noise to speak of): log2(QP) ~ 435 <= 438, the
    HE-standard 128-bit bound for n = 16384 with a ternary secret.
    60 limb transforms per key switch instead of 70 with 30-bit primes,
    K = 4, dnum = 3. Measured on B200 (tools/noise_margin.py):
    decryption margin 27.4 bits (30-bit K=4 dnum=3: 37.7; K=4 dnum=2: 9.4,
    rejected), 134.7 vs 125.4 images/s."""
    return make_params(16384, L=10, T=5, K=5, dnum=2, bits=29, seed=seed)


def lola_cifar_params(seed: int | None = None) -> BfvParams:
    """Config 4: n = 16384, 6 plaintext primes (final bound 183
    bits), L = 6 (its second window stage and 4075-value square add ~25 bits
    of noise over LoLa-MNIST), K = 1, dnum = 6: log2(QP) = 420 <= 438."""
    return make_params(16384, L=6, T=6, K=1, dnum=6, seed=seed)


def lola_cifar_params_w32(seed: int | None = None) -> BfvParams:
    """Config 4 on 29-bit primes (32-bit word kernels, u32 residues: the same
    HBM footprint per ciphertext as the 60-bit set's 6 u64 limbs): L = 11,
    K = 4, dnum = 3 digits of <= 4 primes (P ~ D_j): log2(QP) ~ 435 <= 438.
    Measured on B200 (tools/noise_margin.py): decryption margin 49.0 bits,
    0.27 vs 0.18 images/s for the 60-bit set; (10, 5, 2) is as fast with
    19.0 bits of margin."""
    return make_params(16384, L=11, T=6, K=4, dnum=3, bits=29, seed=seed)


def lola_small_params(seed: int | None = None) -> BfvParams:
    """Config 3: n = 8192, 2 plaintext primes, depth 1 (one square). 54-bit
    primes so that log2(QP) = 216 <= 218, the 128-bit bound at n = 8192:
    L = 3, K = 1, dnum = 3. Measured decryption margin 29.7 bits."""
    return make_params(8192, L=3, T=2, K=1, dnum=3, bits=54, seed=seed)


def lola_small_params_w32(seed: int | None = None) -> BfvParams:
    """Config 3 on 30-bit primes: L = 5, K = 2, dnum = 3 digits of <= 2:
    log2(QP) = 210 <= 218. Measured decryption margin 18.4 bits (L = 6,
    K = 1, dnum = 6: 47.5 bits but 30% slower; dnum = 2 with K = 1 fails)."""
    return make_params(8192, L=5, T=2, K=2, dnum=3, bits=30, seed=seed)
