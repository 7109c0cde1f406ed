"""Ciphertext-level host API over the C-ABI (include/lola_b200.h, §BFV).

Ciphertexts and plaintext operands are torch CUDA tensors of the context's
residue word (`BfvContext.res_dtype`): int32 when every ciphertext and
special prime is below 2^30 (the 32-bit word kernels), else int64:
    ciphertext batch   [count][2][L][n]  (count = B * T, message-major)
    message batch      [B][T][2][L][n]
    plaintext operand  [T][L][n]
Slot values, decrypted residues and keys are int64.
Every method raises on a nonzero C-ABI status; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as nat
from .context import Context, _stream_ptr
from .params import BfvParams

LB_FRESH_IDS = 2**64 - 1  # include/lola_b200.h


class _DevPtr:
    """Exposes a raw device pointer through __cuda_array_interface__."""

    def __init__(self, ptr: int, shape: tuple, dtype="<i8"):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": dtype, "data": (ptr, False), "version": 3,
                                         "strides": None}


def _ptr(t: torch.Tensor, dtype=torch.int64) -> int:
    if not (t.is_cuda and t.is_contiguous() and t.dtype == dtype):
        raise ValueError(f"expected a contiguous {dtype} CUDA tensor")
    return t.data_ptr()


class BfvContext(Context):
    def __init__(self, params: BfvParams):
        super().__init__(params)
        self.L, self.K, self.T = len(params.q), len(params.p), len(params.t)
        self.M = len(params.b)
        self.dnum = params.dnum or self.L
        rb = C.c_uint32()
        nat.call("lb_context_residue_bytes", self.handle, C.byref(rb))
        self.res_dtype = torch.int32 if rb.value == 4 else torch.int64

    # ---- shapes ---------------------------------------------------------------
    def ct_shape(self, count: int) -> tuple:
        return (count, 2, self.L, self.n)

    def empty_cts(self, count: int) -> torch.Tensor:
        return torch.empty(self.ct_shape(count), dtype=self.res_dtype, device="cuda")

    def _r(self, t: torch.Tensor) -> int:
        """Device pointer of a residue tensor (ciphertexts, plaintext operands)."""
        return _ptr(t, self.res_dtype)

    def _count(self, ct: torch.Tensor) -> int:
        per = 2 * self.L * self.n
        if ct.numel() % per:
            raise ValueError("tensor is not a whole number of ciphertexts")
        return ct.numel() // per

    # ---- encode / encrypt / decrypt ------------------------------------------
    def encrypt_slots(self, values: torch.Tensor, id_base: int | None = None, stream=None) -> torch.Tensor:
        """id_base None: fresh randomness ids from the context's counter
        (LB_FRESH_IDS); an explicit id_base is for oracle parity tests."""
        if id_base is None:
            id_base = LB_FRESH_IDS
        values = values.reshape(-1, self.n).contiguous()
        B = values.shape[0]
        out = torch.empty((B, self.T, 2, self.L, self.n), dtype=self.res_dtype, device="cuda")
        nat.call("lb_encrypt_slots", self.handle, _ptr(values), B, id_base, self._r(out), _stream_ptr(stream))
        return out

    def decrypt_slots(self, ct: torch.Tensor, stream=None) -> torch.Tensor:
        B = self._count(ct) // self.T
        out = torch.empty((B, self.T, self.n), dtype=torch.int64, device="cuda")
        nat.call("lb_decrypt_slots", self.handle, self._r(ct), B, _ptr(out), _stream_ptr(stream))
        return out

    def decrypt_coeffs(self, ct: torch.Tensor, stream=None) -> torch.Tensor:
        B = self._count(ct) // self.T
        out = torch.empty((B, self.T, self.n), dtype=torch.int64, device="cuda")
        nat.call("lb_decrypt_coeffs", self.handle, self._r(ct), B, _ptr(out), _stream_ptr(stream))
        return out

    def encode_plain(self, values: torch.Tensor, mul: bool = True, add: bool = True, stream=None):
        values = values.reshape(self.n).contiguous()
        shape = (self.T, self.L, self.n)
        pm = torch.empty(shape, dtype=self.res_dtype, device="cuda") if mul else None
        pa = torch.empty(shape, dtype=self.res_dtype, device="cuda") if add else None
        nat.call("lb_encode_plain", self.handle, _ptr(values), pm.data_ptr() if mul else None,
                 pa.data_ptr() if add else None, _stream_ptr(stream))
        return pm, pa

    # ---- ciphertext ops --------------------------------------------------------
    def _unary(self, name, a, *extra, out=None, stream=None):
        out = torch.empty_like(a) if out is None else out
        nat.call(name, self.handle, self._r(a), *extra, self._r(out), self._count(a), _stream_ptr(stream))
        return out

    def add(self, a, b, out=None, stream=None):
        out = torch.empty_like(a) if out is None else out
        nat.call("lb_ct_add", self.handle, self._r(a), self._r(b), self._r(out), self._count(a), _stream_ptr(stream))
        return out

    def mul_scalar(self, a, s: int, out=None, stream=None):
        return self._unary("lb_ct_mul_scalar", a, int(s), out=out, stream=stream)

    def mul_plain(self, a, pt_mul, out=None, stream=None):
        return self._unary("lb_ct_mul_plain", a, self._r(pt_mul), out=out, stream=stream)

    def add_plain(self, a, pt_add, out=None, stream=None):
        return self._unary("lb_ct_add_plain", a, self._r(pt_add), out=out, stream=stream)

    def rotate(self, a, galois: int, out=None, stream=None):
        return self._unary("lb_ct_rotate", a, int(galois), out=out, stream=stream)

    def mul(self, a, b, out=None, stream=None):
        out = torch.empty_like(a) if out is None else out
        nat.call("lb_ct_mul", self.handle, self._r(a), self._r(b), self._r(out), self._count(a), _stream_ptr(stream))
        return out

    # ---- keys / raw pieces ------------------------------------------------------
    def keygen(self, key_id: int, stream=None) -> None:
        nat.call("lb_keygen", self.handle, key_id, _stream_ptr(stream))

    def key(self, key_id: int) -> torch.Tensor:
        """Copy of the device key [dnum][2][L+K][n] (NTT domain)."""
        p = C.c_void_p()
        nat.call("lb_key_pointer", self.handle, key_id, C.byref(p))
        shape = (self.dnum, 2, self.L + self.K, self.n)
        return torch.as_tensor(_DevPtr(p.value, shape), device="cuda").clone()

    def automorphism(self, a: torch.Tensor, galois: int, limbs: int, stream=None) -> torch.Tensor:
        out = torch.empty_like(a)
        polys = a.numel() // (limbs * self.n)
        nat.call("lb_automorphism", self.handle, self._r(a), self._r(out), polys, limbs, galois, _stream_ptr(stream))
        return out

    def key_switch(self, d: torch.Tensor, key_id: int, stream=None):
        count = d.numel() // (self.L * self.n)
        u0, u1 = torch.empty_like(d), torch.empty_like(d)
        nat.call("lb_key_switch", self.handle, self._r(d), key_id, self._r(u0), self._r(u1), count,
                 _stream_ptr(stream))
        return u0, u1


def galois_exponent_columns(n: int, k: int) -> int:
    """Right shift of both slot rows by k (reference ring.cpp:173-182)."""
    if not 0 <= k < n // 2:
        raise ValueError("k out of range")
    return int(nat.lib().lb_galois_exponent_columns(n, k))


def galois_exponent_rows(n: int) -> int:
    return int(nat.lib().lb_galois_exponent_rows(n))
