"""ctypes binding of oracle/_ref/libbfvoracle.so (our CPU BFV-RNS restatement).

TEST INFRASTRUCTURE ONLY — the ciphertext-level checker (see bfv_oracle.h for
its parity status). Ciphertexts are numpy uint64 arrays [2][L][n] of
COEFFICIENTS.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB = Path(__file__).resolve().parent / "_ref" / "libbfvoracle.so"
u32, u64, i64 = C.c_uint32, C.c_uint64, C.c_int64
P64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)

_lib = None


def lib():
    global _lib
    if _lib is None:
        l = C.CDLL(str(LIB))
        l.bo_create.restype = C.c_void_p
        l.bo_create.argtypes = [u32, P64, u32, P64, u32, P64, u32, P64, u32, u32, u64]
        l.bo_destroy.argtypes = [C.c_void_p]
        l.bo_last_error.restype = C.c_char_p
        l.bo_prng.restype = u64
        l.bo_prng.argtypes = [u64, u64, u64]
        sigs = {
            "bo_secret": [C.c_void_p, PI64],
            "bo_slot_encode": [C.c_void_p, u32, P64, P64],
            "bo_slot_decode": [C.c_void_p, u32, P64, P64],
            "bo_encrypt": [C.c_void_p, u32, P64, u64, P64],
            "bo_decrypt": [C.c_void_p, u32, P64, P64],
            "bo_mul_plain": [C.c_void_p, u32, P64, P64, P64],
            "bo_add_plain": [C.c_void_p, u32, P64, P64, P64],
            "bo_mul_scalar": [C.c_void_p, P64, i64, P64],
            "bo_add": [C.c_void_p, P64, P64, P64],
            "bo_galois_key": [C.c_void_p, u64, P64],
            "bo_rotate": [C.c_void_p, P64, u64, P64],
            "bo_time_rotate": [C.c_void_p, P64, u64, u32, P64, C.POINTER(C.c_double)],
            "bo_mul": [C.c_void_p, u32, P64, P64, P64],
            "bo_phase": [C.c_void_p, P64, P64],
        }
        for k, v in sigs.items():
            f = getattr(l, k)
            f.argtypes = v
            f.restype = C.c_int
        _lib = l
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(P64)


def _u(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def prng(seed: int, stream: int, index: int) -> int:
    return int(lib().bo_prng(seed, stream, index))


class Oracle:
    def __init__(self, n, q, p, b, t, dnum=0, seed=0):
        self.n, self.L, self.K, self.M, self.T = n, len(q), len(p), len(b), len(t)
        self.q, self.p, self.b, self.t = list(q), list(p), list(b), list(t)
        self.dnum = dnum or len(q)
        arrs = [_u(x) if len(x) else np.zeros(1, np.uint64) for x in (q, p, b, t)]
        self._keep = arrs
        self.h = lib().bo_create(n, _p(arrs[0]), len(q), _p(arrs[1]), len(p), _p(arrs[2]), len(b), _p(arrs[3]),
                                 len(t), dnum, seed)
        if not self.h:
            raise RuntimeError(lib().bo_last_error().decode())

    @classmethod
    def from_params(cls, prm):
        return cls(prm.n, prm.q, prm.p, prm.b, prm.t, prm.dnum, prm.seed)

    def __del__(self):
        if getattr(self, "h", None):
            lib().bo_destroy(self.h)
            self.h = None

    def _chk(self, rc):
        if rc:
            raise RuntimeError(lib().bo_last_error().decode())

    def _ct(self):
        return np.zeros((2, self.L, self.n), dtype=np.uint64)

    def secret(self) -> np.ndarray:
        s = np.zeros(self.n, dtype=np.int64)
        self._chk(lib().bo_secret(self.h, s.ctypes.data_as(PI64)))
        return s

    def slot_encode(self, tj, slots):
        s = _u(slots)
        out = np.zeros(self.n, np.uint64)
        self._chk(lib().bo_slot_encode(self.h, tj, _p(s), _p(out)))
        return out

    def slot_decode(self, tj, coeffs):
        c = _u(coeffs)
        out = np.zeros(self.n, np.uint64)
        self._chk(lib().bo_slot_decode(self.h, tj, _p(c), _p(out)))
        return out

    def encrypt(self, tj, m_coeffs, ct_id):
        m = _u(m_coeffs)
        out = self._ct()
        self._chk(lib().bo_encrypt(self.h, tj, _p(m), ct_id, _p(out)))
        return out

    def decrypt(self, tj, ct):
        c = _u(ct)
        out = np.zeros(self.n, np.uint64)
        self._chk(lib().bo_decrypt(self.h, tj, _p(c), _p(out)))
        return out

    def mul_plain(self, tj, ct, slots):
        c, s = _u(ct), _u(slots)
        out = self._ct()
        self._chk(lib().bo_mul_plain(self.h, tj, _p(c), _p(s), _p(out)))
        return out

    def add_plain(self, tj, ct, slots):
        c, s = _u(ct), _u(slots)
        out = self._ct()
        self._chk(lib().bo_add_plain(self.h, tj, _p(c), _p(s), _p(out)))
        return out

    def mul_scalar(self, ct, s):
        c = _u(ct)
        out = self._ct()
        self._chk(lib().bo_mul_scalar(self.h, _p(c), int(s), _p(out)))
        return out

    def add(self, a, b):
        a, b = _u(a), _u(b)
        out = self._ct()
        self._chk(lib().bo_add(self.h, _p(a), _p(b), _p(out)))
        return out

    def galois_key(self, g):
        out = np.zeros((self.dnum, 2, self.L + self.K, self.n), np.uint64)
        self._chk(lib().bo_galois_key(self.h, g, _p(out)))
        return out

    def rotate(self, ct, g):
        c = _u(ct)
        out = self._ct()
        self._chk(lib().bo_rotate(self.h, _p(c), g, _p(out)))
        return out

    def time_rotate(self, ct, g, reps: int = 1) -> tuple[np.ndarray, float]:
        """(rotated ciphertext, seconds for `reps` rotations), key made once."""
        c = _u(ct)
        out = self._ct()
        sec = C.c_double()
        self._chk(lib().bo_time_rotate(self.h, _p(c), g, reps, _p(out), C.byref(sec)))
        return out, sec.value

    def mul(self, tj, a, b):
        a, b = _u(a), _u(b)
        out = self._ct()
        self._chk(lib().bo_mul(self.h, tj, _p(a), _p(b), _p(out)))
        return out

    def phase(self, ct) -> np.ndarray:
        c = _u(ct)
        out = np.zeros((self.L, self.n), np.uint64)
        self._chk(lib().bo_phase(self.h, _p(c), _p(out)))
        return out

    def noise_bits(self, tj, ct, m_coeffs) -> float:
        """log2 of max |c0 + c1 s - round(Q m / t)| centered mod Q (exact)."""
        import math

        x = self.phase(ct)
        Q = 1
        for qi in self.q:
            Q *= qi
        t = self.t[tj]
        coef = [(Q // qi) * pow(Q // qi, -1, qi) for qi in self.q]
        worst = 0
        cols = [x[i].tolist() for i in range(self.L)]
        for k in range(self.n):
            v = sum(cols[i][k] * coef[i] for i in range(self.L)) % Q
            e = (v - (Q * int(m_coeffs[k]) + t // 2) // t) % Q
            if e > Q // 2:
                e -= Q
            worst = max(worst, abs(e))
        return math.log2(worst) if worst else 0.0
