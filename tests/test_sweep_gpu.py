"""BASELINE config 1 (HE primitive sweep) parity: n in {4096..32768} with
2..12 ciphertext limbs. Every limb transform against the reference's
NttTables; ct x pt, ct + ct, rotations (steps 1, 2, 4, ..., n/4 and the row
swap) and square + relinearize against the CPU BFV oracle, coefficient by
coefficient; decryptions against the reference ring ops."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import refbind as R
from oracle.bfvbind import Oracle
from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns, galois_exponent_rows
from paper_1812_10659_b200.context import bitrev_perm
from paper_1812_10659_b200.params import make_params

pytestmark = pytest.mark.gpu

SWEEP = [(4096, 2), (4096, 12), (8192, 8), (16384, 4), (16384, 12), (32768, 2), (32768, 8)]
# 30-bit primes: the 32-bit word transforms
SWEEP32 = [(4096, 12), (16384, 14), (32768, 6)]


def coeffs(cx, ct):
    x = ct.reshape(-1, 2, cx.L, cx.n).to(torch.int64, copy=True)  # residue words -> the NTT engine's u64 limbs
    cx.ntt_inverse(x, limbs=cx.L)
    torch.cuda.synchronize()
    return x.cpu().numpy().astype(np.uint64)


@pytest.mark.parametrize("n,L", SWEEP, ids=[f"n{n}_L{L}" for n, L in SWEEP])
def test_ntt_every_limb_matches_reference(n, L):
    prm = make_params(n, L=L, T=1, K=1, seed=n + L)
    cx = BfvContext(prm)
    primes = cx.primes
    rng = np.random.default_rng(n * 31 + L)
    polys = 3
    data = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes]) for _ in range(polys)])
    dev = torch.from_numpy(data.astype(np.int64)).cuda()
    cx.ntt_forward(dev, limbs=len(primes))
    torch.cuda.synchronize()
    got = dev.cpu().numpy().astype(np.uint64)
    br = bitrev_perm(n)
    for i, p in enumerate(primes):
        assert np.array_equal(got[1, i][br], R.ntt_forward(p, data[1, i])), f"limb {i} (p={p})"
    cx.ntt_inverse(dev, limbs=len(primes))
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().astype(np.uint64), data)


@pytest.mark.parametrize("n,L", SWEEP32, ids=[f"w32_n{n}_L{L}" for n, L in SWEEP32])
def test_ntt_word32_matches_reference(n, L):
    prm = make_params(n, L=L, T=1, K=1, bits=30, seed=n + L)
    cx = BfvContext(prm)
    primes = cx.primes
    assert all(p < 1 << 30 for p in primes[:L])
    rng = np.random.default_rng(n * 37 + L)
    data = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes]) for _ in range(2)])
    dev = torch.from_numpy(data.astype(np.int64)).cuda()
    cx.ntt_forward(dev, limbs=len(primes))
    torch.cuda.synchronize()
    got = dev.cpu().numpy().astype(np.uint64)
    br = bitrev_perm(n)
    for i, p in enumerate(primes):
        assert np.array_equal(got[0, i][br], R.ntt_forward(p, data[0, i])), f"limb {i} (p={p})"
    cx.ntt_inverse(dev, limbs=len(primes))
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().astype(np.uint64), data)


@pytest.mark.parametrize("n,L,K,dnum,bits", [(4096, 12, 1, 0, 60), (16384, 4, 1, 0, 60), (32768, 2, 1, 0, 60),
                                              (32768, 6, 1, 0, 60), (32768, 12, 2, 6, 60), (32768, 8, 4, 2, 29),
                                              (8192, 12, 4, 3, 29)],
                         ids=["n4096_L12", "n16384_L4", "n32768_L2", "n32768_L6", "n32768_L12_K2_dnum6",
                              "w32_n32768_L8_K4_dnum2", "w32_n8192_L12_K4_dnum3"])
def test_ciphertext_primitives_match_oracle(n, L, K, dnum, bits):
    """60-bit sets on the 64-bit kernels; 29-bit sets on the 32-bit word
    kernels with u32 residue storage (n = 32768: eight-CTA clusters)."""
    prm = make_params(n, L=L, T=1, K=K, dnum=dnum, bits=bits, seed=3 * n + L)
    cx = BfvContext(prm)
    o = Oracle.from_params(prm)
    t = prm.t[0]
    rng = np.random.default_rng(L)
    vals = rng.integers(-5000, 5000, size=(2, n), dtype=np.int64)
    ct = cx.encrypt_slots(torch.from_numpy(vals).cuda(), id_base=500)
    A = coeffs(cx, ct)
    m = [R.slot_encode(t, np.mod(v, t).astype(np.uint64)) for v in vals]
    for c in range(2):
        assert np.array_equal(A[c], o.encrypt(0, m[c], 500 + c))
    w = rng.integers(-100, 100, size=n, dtype=np.int64)
    pm, _ = cx.encode_plain(torch.from_numpy(w).cuda(), add=False)
    got = coeffs(cx, cx.mul_plain(ct, pm))
    wt = np.mod(w, t).astype(np.uint64)
    assert np.array_equal(got[0], o.mul_plain(0, A[0], wt))
    got = coeffs(cx, cx.add(ct[:1], ct[1:]))
    assert np.array_equal(got[0], o.add(A[0], A[1]))
    steps = [1 << i for i in range(0, (n // 4).bit_length(), max(1, ((n // 4).bit_length()) // 3))]
    for k in [*steps[:3], n // 4]:
        g = galois_exponent_columns(n, k)
        r = coeffs(cx, cx.rotate(ct[:1], g))
        assert np.array_equal(r[0], o.rotate(A[0], g)), f"rotation by {k}"
    g = galois_exponent_rows(n)
    r = cx.rotate(ct[:1], g)
    assert np.array_equal(coeffs(cx, r)[0], o.rotate(A[0], g))
    assert np.array_equal(cx.decrypt_coeffs(r).cpu().numpy()[0, 0].astype(np.uint64), R.galois_apply(t, m[0], g))
    sq = cx.mul(ct[:1], ct[:1])
    assert np.array_equal(coeffs(cx, sq)[0], o.mul(0, A[0], A[0]))
    assert np.array_equal(cx.decrypt_coeffs(sq).cpu().numpy()[0, 0].astype(np.uint64), R.poly_mul(t, m[0], m[0]))
