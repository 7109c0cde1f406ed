"""Ciphertext-level parity: every device BFV primitive against the CPU BFV
oracle (oracle/bfv_oracle.cpp) coefficient by coefficient, and the decrypted
results against the reference ring semantics (oracle/_ref/libpackref.so)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import refbind as R
from oracle.bfvbind import Oracle
from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns, galois_exponent_rows
from paper_1812_10659_b200.params import make_params

pytestmark = pytest.mark.gpu


# 60-bit primes run the 64-bit word kernels; 30-bit primes (< 2^30) the
# 32-bit word NTT / key-switch kernels with u32 residue storage, with 1-, 3-,
# 4- and 5-prime digits (the last: the lola-mnist default digit structure).
@pytest.fixture(scope="module", params=[(4096, 3, 2, 1, 0, 60), (8192, 4, 1, 1, 0, 60), (4096, 5, 2, 2, 3, 60),
                                        (4096, 6, 2, 3, 2, 30), (8192, 10, 2, 4, 3, 30), (4096, 4, 1, 1, 4, 30),
                                        (8192, 10, 2, 5, 2, 29)],
                ids=["n4096_L3_T2", "n8192_L4_T1", "n4096_L5_K2_dnum3", "w32_n4096_L6_K3_dnum2",
                     "w32_n8192_L10_K4_dnum3", "w32_n4096_L4_K1", "w32_n8192_L10_K5_dnum2"])
def env(request):
    n, L, T, K, dnum, bits = request.param
    prm = make_params(n, L=L, T=T, K=K, dnum=dnum, bits=bits, seed=11)
    cx = BfvContext(prm)
    o = Oracle.from_params(prm)
    return prm, cx, o


def coeffs(cx, ct: torch.Tensor) -> np.ndarray:
    """Device ciphertexts (evaluation domain) -> coefficient numpy [count][2][L][n]."""
    x = ct.reshape(-1, 2, cx.L, cx.n).to(torch.int64, copy=True)  # residue words -> the NTT engine's u64 limbs
    cx.ntt_inverse(x, limbs=cx.L)
    torch.cuda.synchronize()
    return x.cpu().numpy().astype(np.uint64)


def rand_values(prm, B, lo=-1000, hi=1000, seed=0):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=(B, prm.n), dtype=np.int64)


def encrypt(cx, prm, vals, id_base=100):
    return cx.encrypt_slots(torch.from_numpy(vals).cuda(), id_base=id_base)


def plain_m(prm, tj, vals_row):
    t = prm.t[tj]
    return R.slot_encode(t, np.mod(vals_row, t).astype(np.uint64))


def test_encrypt_matches_oracle(env):
    prm, cx, o = env
    vals = rand_values(prm, 2)
    ct = encrypt(cx, prm, vals)
    got = coeffs(cx, ct)
    for b in range(2):
        for tj in range(cx.T):
            c = b * cx.T + tj
            want = o.encrypt(tj, plain_m(prm, tj, vals[b]), 100 + c)
            assert np.array_equal(got[c], want), f"ciphertext {c} differs"


def test_decrypt_roundtrip(env):
    prm, cx, o = env
    vals = rand_values(prm, 3, seed=1)
    ct = encrypt(cx, prm, vals)
    slots = cx.decrypt_slots(ct).cpu().numpy()
    m = cx.decrypt_coeffs(ct).cpu().numpy().astype(np.uint64)
    got = coeffs(cx, ct)
    for b in range(3):
        for tj, t in enumerate(prm.t):
            assert np.array_equal(slots[b, tj], np.mod(vals[b], t))
            assert np.array_equal(m[b, tj], o.decrypt(tj, got[b * cx.T + tj]))


def test_elementwise_ops(env):
    prm, cx, o = env
    vals = rand_values(prm, 2, seed=2)
    w = rand_values(prm, 1, seed=3)[0]
    a = encrypt(cx, prm, vals, 7)
    b = encrypt(cx, prm, vals[::-1].copy(), 9)
    A, Bc = coeffs(cx, a), coeffs(cx, b)
    pm, pa = cx.encode_plain(torch.from_numpy(w).cuda())
    s_add = coeffs(cx, cx.add(a, b))
    s_sc = coeffs(cx, cx.mul_scalar(a, -45))
    s_mp = coeffs(cx, cx.mul_plain(a, pm))
    s_ap = coeffs(cx, cx.add_plain(a, pa))
    for c in range(2 * cx.T):
        tj = c % cx.T
        wt = np.mod(w, prm.t[tj]).astype(np.uint64)
        assert np.array_equal(s_add[c], o.add(A[c], Bc[c]))
        assert np.array_equal(s_sc[c], o.mul_scalar(A[c], -45))
        assert np.array_equal(s_mp[c], o.mul_plain(tj, A[c], wt))
        assert np.array_equal(s_ap[c], o.add_plain(tj, A[c], wt))


def test_galois_key_matches_oracle(env):
    prm, cx, o = env
    g = galois_exponent_columns(prm.n, 1)
    cx.keygen(g)
    k = cx.key(g)
    kc = k.clone()
    cx.ntt_inverse(kc, limbs=cx.L + cx.K)
    torch.cuda.synchronize()
    assert np.array_equal(kc.cpu().numpy().astype(np.uint64), o.galois_key(g))


@pytest.mark.parametrize("k", [1, 2, 7, "rows"])
def test_rotate_matches_oracle_and_reference(env, k):
    prm, cx, o = env
    n = prm.n
    g = galois_exponent_rows(n) if k == "rows" else galois_exponent_columns(n, k)
    assert g == (R.galois_exponent_rows(n) if k == "rows" else R.galois_exponent_columns(n, k))
    vals = rand_values(prm, 1, seed=4)
    a = encrypt(cx, prm, vals, 3)
    A = coeffs(cx, a)
    r = cx.rotate(a, g)
    got = coeffs(cx, r)
    m = cx.decrypt_coeffs(r).cpu().numpy().astype(np.uint64)
    for tj, t in enumerate(prm.t):
        assert np.array_equal(got[tj], o.rotate(A[tj], g))
        assert np.array_equal(m[0, tj], R.galois_apply(t, plain_m(prm, tj, vals[0]), g))


def test_mul_matches_oracle_and_reference(env):
    prm, cx, o = env
    vals = rand_values(prm, 1, seed=5)
    vals2 = rand_values(prm, 1, seed=6)
    a = encrypt(cx, prm, vals, 21)
    b = encrypt(cx, prm, vals2, 23)
    A, Bc = coeffs(cx, a), coeffs(cx, b)
    prod = cx.mul(a, b)
    sq = cx.mul(a, a)
    got_p, got_s = coeffs(cx, prod), coeffs(cx, sq)
    mp = cx.decrypt_coeffs(prod).cpu().numpy().astype(np.uint64)
    for tj, t in enumerate(prm.t):
        assert np.array_equal(got_p[tj], o.mul(tj, A[tj], Bc[tj]))
        assert np.array_equal(got_s[tj], o.mul(tj, A[tj], A[tj]))
        want = R.poly_mul(t, plain_m(prm, tj, vals[0]), plain_m(prm, tj, vals2[0]))
        assert np.array_equal(mp[0, tj], want)


def test_tmem_accumulator_variant_matches_oracle():
    """The TMEM-accumulator key-switch kernel (LB_KS_TMEM=1) is bit-exact too."""
    import subprocess
    import sys

    code = (
        "import sys; sys.path.insert(0, '.');"
        "import numpy as np, torch;"
        "from oracle.bfvbind import Oracle;"
        "from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns;"
        "from paper_1812_10659_b200.params import make_params;"
        "prm = make_params(16384, L=5, T=1, K=1, seed=4); cx = BfvContext(prm); o = Oracle.from_params(prm);"
        "v = torch.arange(prm.n, dtype=torch.int64, device='cuda').reshape(1, -1) - 77;"
        "ct = cx.encrypt_slots(v, id_base=9); g = galois_exponent_columns(prm.n, 5);"
        "c = lambda t: (lambda x: (cx.ntt_inverse(x, limbs=prm.L), torch.cuda.synchronize(), x.cpu().numpy().astype(np.uint64))[2])(t.reshape(-1, 2, prm.L, prm.n).clone());"
        "assert np.array_equal(c(cx.rotate(ct, g))[0], o.rotate(c(ct)[0], g));"
        "print('ok')"
    )
    import os

    env = dict(os.environ, LB_KS_TMEM="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
