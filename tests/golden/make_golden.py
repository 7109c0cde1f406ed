"""Regenerates tests/golden/ring_vectors.json from the reference (packnn,
compiled in place into oracle/_ref/libpackref.so). Run in the dev container
(needs /root/reference to build the library); the JSON is committed so the
checks also run where the reference is absent.

Each case: a seeded input (SplitMix64, paper_1812_10659_b200.nets.splitmix64),
the reference's output digest (sha256 of the little-endian u64 array) and
its first 8 values.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import refbind as R  # noqa: E402
from paper_1812_10659_b200.nets import splitmix64  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def rand_mod(seed: int, n: int, p: int) -> np.ndarray:
    return (splitmix64(seed, n) % np.uint64(p)).astype(np.uint64)


def main() -> None:
    cases = []
    # one 60-bit ciphertext prime (== 1 mod 2^16) and the reference's plaintext primes
    primes = [1152921504606584833, 2148728833, 2281701377]
    for n in (4096, 8192, 16384):
        for p in primes:
            if (p - 1) % (2 * n):
                continue
            a = rand_mod(1000 + n + p % 97, n, p)
            b = rand_mod(2000 + n + p % 89, n, p)
            s = rand_mod(3000 + n + p % 83, n, p)
            fwd = R.ntt_forward(p, a)
            out = {
                "n": n, "p": p, "psi": R.root_of_unity(p, 2 * n),
                "seeds": {"a": 1000 + n + p % 97, "b": 2000 + n + p % 89, "slots": 3000 + n + p % 83},
                "ntt_forward": {"sha256": digest(fwd), "head": [int(v) for v in fwd[:8]]},
                "poly_mul": {"sha256": digest(R.poly_mul(p, a, b))},
                "galois_col1": {"g": R.galois_exponent_columns(n, 1),
                                "sha256": digest(R.galois_apply(p, a, R.galois_exponent_columns(n, 1)))},
                "galois_rows": {"g": R.galois_exponent_rows(n),
                                "sha256": digest(R.galois_apply(p, a, R.galois_exponent_rows(n)))},
                "slot_encode": {"sha256": digest(R.slot_encode(p, s))},
            }
            cases.append(out)
    kat = {
        # proj/tests/test_ring.cpp:45-56, 58-70, 126-141, 176-186
        "negacyclic_17_n4": {"a": [1, 2, 3, 4], "b": [5, 6, 7, 8], "p": 17,
                             "want": [int(v) for v in R.poly_mul(17, [1, 2, 3, 4], [5, 6, 7, 8])]},
        "wraparound_97_n8": [int(v) for v in R.poly_mul(97, [0] * 7 + [1], [0, 1] + [0] * 6)],
        "crt_5_7": R.crt_join_center([2, 3], [5, 7], center=False),
    }
    path = Path(__file__).with_name("ring_vectors.json")
    path.write_text(json.dumps({"generator": "tests/golden/make_golden.py", "cases": cases, "kat": kat}, indent=1))
    print(f"wrote {path} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
