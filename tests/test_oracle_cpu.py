"""The CPU oracles, pinned: the compiled reference against its own
known-answer tests (proj/tests/test_ring.cpp) and the committed golden
vectors; the BFV oracle against the reference ring semantics."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import refbind as R
from oracle.bfvbind import Oracle
from paper_1812_10659_b200.nets import splitmix64
from paper_1812_10659_b200.params import make_params

GOLD = json.loads((Path(__file__).parent / "golden" / "ring_vectors.json").read_text())


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def rand_mod(seed, n, p):
    return (splitmix64(seed, n) % np.uint64(p)).astype(np.uint64)


def test_reference_known_answers():
    # proj/tests/test_ring.cpp:45-56: (1+2x+3x^2+4x^3)(5+6x+7x^2+8x^3) mod (x^4+1, 17)
    assert R.poly_mul(17, [1, 2, 3, 4], [5, 6, 7, 8]).tolist() == [12, 15, 2, 9]
    assert R.schoolbook_mul(17, [1, 2, 3, 4], [5, 6, 7, 8]).tolist() == [12, 15, 2, 9]
    # :58-70 x^7 * x = -1 (p = 97)
    assert R.poly_mul(97, [0] * 7 + [1], [0, 1] + [0] * 6).tolist() == [96] + [0] * 7
    # :19-29 root search
    w = R.root_of_unity(17, 8)
    assert pow(w, 8, 17) == 1 and pow(w, 4, 17) == 16 and R.root_of_unity(17, 2) == 16
    # :126-141 rotations at n = 4: (1,2,3,4) -> columns(1) (2,1,4,3), rows (3,4,1,2)
    enc = R.slot_encode(17, [1, 2, 3, 4])
    assert R.slot_decode(17, R.galois_apply(17, enc, R.galois_exponent_columns(4, 1))).tolist() == [2, 1, 4, 3]
    assert R.slot_decode(17, R.galois_apply(17, enc, R.galois_exponent_rows(4))).tolist() == [3, 4, 1, 2]
    # :176-186 CRT
    assert R.crt_join_center([2, 3], [5, 7], center=False) == 17
    assert R.crt_join_center([3, 4], [5, 7], center=True) == 18 - 35
    assert GOLD["kat"]["negacyclic_17_n4"]["want"] == [12, 15, 2, 9]
    assert GOLD["kat"]["crt_5_7"] == 17


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"n{c['n']}-p{c['p']}")
def test_reference_reproduces_golden(case):
    n, p, sd = case["n"], case["p"], case["seeds"]
    a, b, s = rand_mod(sd["a"], n, p), rand_mod(sd["b"], n, p), rand_mod(sd["slots"], n, p)
    assert R.root_of_unity(p, 2 * n) == case["psi"]
    fwd = R.ntt_forward(p, a)
    assert digest(fwd) == case["ntt_forward"]["sha256"] and fwd[:8].tolist() == case["ntt_forward"]["head"]
    assert digest(R.poly_mul(p, a, b)) == case["poly_mul"]["sha256"]
    assert digest(R.galois_apply(p, a, case["galois_col1"]["g"])) == case["galois_col1"]["sha256"]
    assert digest(R.slot_encode(p, s)) == case["slot_encode"]["sha256"]
    assert np.array_equal(R.ntt_inverse(p, fwd), a)


@pytest.mark.parametrize("case", [c for c in GOLD["cases"] if c["p"] < 2**32 and c["n"] <= 8192],
                         ids=lambda c: f"n{c['n']}-t{c['p']}")
def test_bfv_oracle_plaintext_side_matches_golden(case):
    n, t = case["n"], case["p"]
    prm = make_params(n, L=2, T=1, K=1, plain=[t])
    o = Oracle.from_params(prm)
    s = rand_mod(case["seeds"]["slots"], n, t)
    assert digest(o.slot_encode(0, s)) == case["slot_encode"]["sha256"]
    assert np.array_equal(o.slot_decode(0, o.slot_encode(0, s)), s)


@pytest.fixture(scope="module")
def small():
    prm = make_params(4096, L=4, T=2, K=1, seed=7)
    return prm, Oracle.from_params(prm)


def test_bfv_oracle_ops_decrypt_to_reference_ring_ops(small):
    prm, o = small
    n = prm.n
    rng = np.random.default_rng(3)
    for tj, t in enumerate(prm.t):
        m = R.slot_encode(t, rng.integers(0, t, n, dtype=np.uint64))
        w = rng.integers(0, t, n, dtype=np.uint64)
        ct = o.encrypt(tj, m, 40 + tj)
        assert np.array_equal(o.decrypt(tj, ct), m)
        assert np.array_equal(o.decrypt(tj, o.mul_plain(tj, ct, w)), R.poly_mul(t, m, R.slot_encode(t, w)))
        assert np.array_equal(o.decrypt(tj, o.add_plain(tj, ct, w)), R.poly_add(t, m, R.slot_encode(t, w)))
        assert np.array_equal(o.decrypt(tj, o.mul_scalar(ct, -5)), R.poly_scale(t, m, t - 5))
        g = R.galois_exponent_columns(n, 3)
        assert np.array_equal(o.decrypt(tj, o.rotate(ct, g)), R.galois_apply(t, m, g))
        assert np.array_equal(o.decrypt(tj, o.mul(tj, ct, ct)), R.poly_mul(t, m, m))


def test_bfv_noise_growth_is_bounded(small):
    prm, o = small
    t = prm.t[0]
    m = R.slot_encode(t, np.arange(prm.n, dtype=np.uint64) % t)
    ct = o.encrypt(0, m, 1)
    fresh = o.noise_bits(0, ct, m)
    rot = o.noise_bits(0, o.rotate(ct, R.galois_exponent_columns(prm.n, 1)), R.galois_apply(t, m, 3 ** (prm.n // 2 - 1) % (2 * prm.n)))
    assert fresh < 6 and rot < 16
