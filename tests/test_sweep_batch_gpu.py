"""BASELINE config 1 at batch: 8 ciphertexts per launch (a 64-ciphertext
batch is exercised by the bench's primitive leg), n in {4096, 8192, 16384,
32768}, on a 60-bit set (64-bit word kernels) and a 29-bit set (32-bit word
kernels, u32 residues). Every ciphertext of the batch is compared with the
CPU BFV oracle coefficient by coefficient after encrypt, ct x pt, ct + ct,
EVERY rotation by k = 2^i (i = 0 .. log2(n/4)) and the row swap
(proj/src/ring.cpp:173-193), and square + relinearize; each rotation's
decryption equals the reference's galois_apply (ring.cpp:155-171). The
oracle calls release the GIL, so they run on a thread pool."""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np
import pytest
import torch

from oracle import refbind as R
from oracle.bfvbind import Oracle
from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns, galois_exponent_rows
from paper_1812_10659_b200.context import bitrev_perm
from paper_1812_10659_b200.params import make_params

pytestmark = pytest.mark.gpu

B = 8
# (n, L, K, dnum, bits)
SETS = [(4096, 4, 1, 0, 60), (8192, 6, 2, 3, 60), (16384, 5, 2, 3, 60), (32768, 4, 1, 0, 60),
        (4096, 6, 2, 3, 29), (8192, 8, 4, 2, 29), (16384, 10, 5, 2, 29), (32768, 8, 4, 2, 29)]
IDS = [f"{'w32' if b < 32 else 'w64'}_n{n}_L{L}_K{K}" for n, L, K, d, b in SETS]
POOL = cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4))


def coeffs(cx, ct):
    x = ct.reshape(-1, 2, cx.L, cx.n).to(torch.int64, copy=True)
    cx.ntt_inverse(x, limbs=cx.L)
    torch.cuda.synchronize()
    return x.cpu().numpy().astype(np.uint64)


def pmap(fn, items):
    return list(POOL.map(fn, items))


@pytest.fixture(scope="module", params=SETS, ids=IDS)
def env(request):
    n, L, K, dnum, bits = request.param
    prm = make_params(n, L=L, T=1, K=K, dnum=dnum, bits=bits, seed=7 * n + L)
    cx = BfvContext(prm)
    assert (cx.res_dtype == torch.int32) == (bits < 30)
    o = Oracle.from_params(prm)
    rng = np.random.default_rng(n + bits)
    vals = rng.integers(-3000, 3000, size=(B, n), dtype=np.int64)
    ct = cx.encrypt_slots(torch.from_numpy(vals).cuda(), id_base=1000)
    A = coeffs(cx, ct)
    return prm, cx, o, vals, ct, A


def test_encrypt_batch(env):
    prm, cx, o, vals, ct, A = env
    t = prm.t[0]
    m = [R.slot_encode(t, np.mod(v, t).astype(np.uint64)) for v in vals]
    want = pmap(lambda b: o.encrypt(0, m[b], 1000 + b), range(B))
    for b in range(B):
        assert np.array_equal(A[b], want[b]), f"ciphertext {b}"


def test_plain_and_add_batch(env):
    prm, cx, o, vals, ct, A = env
    t = prm.t[0]
    w = np.random.default_rng(5).integers(-100, 100, size=prm.n, dtype=np.int64)
    pm, _ = cx.encode_plain(torch.from_numpy(w).cuda(), add=False)
    got = coeffs(cx, cx.mul_plain(ct, pm))
    wt = np.mod(w, t).astype(np.uint64)
    want = pmap(lambda b: o.mul_plain(0, A[b], wt), range(B))
    for b in range(B):
        assert np.array_equal(got[b], want[b]), f"ct x pt {b}"
    rolled = torch.roll(ct, 1, dims=0).contiguous()
    got = coeffs(cx, cx.add(ct, rolled))
    for b in range(B):
        assert np.array_equal(got[b], o.add(A[b], A[(b - 1) % B])), f"ct + ct {b}"


def test_every_rotation_batch(env):
    prm, cx, o, vals, ct, A = env
    n, t = prm.n, prm.t[0]
    amounts = [1 << i for i in range((n // 4).bit_length())]
    assert amounts[-1] == n // 4
    gs = [(f"col {k}", galois_exponent_columns(n, k)) for k in amounts] + [("rows", galois_exponent_rows(n))]
    for name, g in gs:
        r = cx.rotate(ct, g)
        got = coeffs(cx, r)
        want = pmap(lambda b: o.rotate(A[b], g), range(B))
        for b in range(B):
            assert np.array_equal(got[b], want[b]), f"rotation {name}, ciphertext {b}"
        dec = cx.decrypt_coeffs(r).cpu().numpy().astype(np.uint64)
        b = amounts.index(int(name.split()[1])) % B if name != "rows" else B - 1
        m = R.slot_encode(t, np.mod(vals[b], t).astype(np.uint64))
        assert np.array_equal(dec[b, 0], R.galois_apply(t, m, g)), f"decrypted rotation {name}"


def test_square_relin_batch(env):
    prm, cx, o, vals, ct, A = env
    t = prm.t[0]
    sq = cx.mul(ct, ct)
    got = coeffs(cx, sq)
    want = pmap(lambda b: o.mul(0, A[b], A[b]), range(B))
    for b in range(B):
        assert np.array_equal(got[b], want[b]), f"square {b}"
    dec = cx.decrypt_coeffs(sq).cpu().numpy().astype(np.uint64)
    m = R.slot_encode(t, np.mod(vals[3], t).astype(np.uint64))
    assert np.array_equal(dec[3, 0], R.poly_mul(t, m, m))


@pytest.mark.parametrize("n,L", [(4096, 6), (8192, 12), (16384, 10), (32768, 6)])
def test_u32_storage_ntt_matches_reference(n, L):
    """lb_ntt_forward_u32 / lb_ntt_inverse_u32: the u32-storage transforms
    the key switch runs (and the bench's NTT roofline times)."""
    prm = make_params(n, L=L, T=1, K=1, bits=29, seed=n + 3 * L)
    cx = BfvContext(prm)
    primes = prm.q
    rng = np.random.default_rng(n + L)
    data = np.stack([np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes]) for _ in range(B)])
    dev = torch.from_numpy(data.astype(np.int32)).cuda()
    cx.ntt_forward(dev, limbs=L)
    torch.cuda.synchronize()
    got = dev.cpu().numpy().astype(np.uint32).astype(np.uint64)
    br = bitrev_perm(n)
    for b in (0, B - 1):
        for i, p in enumerate(primes):
            assert np.array_equal(got[b, i][br], R.ntt_forward(p, data[b, i])), f"poly {b} limb {i}"
    cx.ntt_inverse(dev, limbs=L)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().astype(np.uint32).astype(np.uint64), data)
