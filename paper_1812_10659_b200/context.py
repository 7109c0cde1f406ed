"""Host-side handle of a device context (include/lola_b200.h: lb_context).

Device memory is plain torch int64 CUDA tensors (values < 2^62, so the
signed view is exact); only their data pointers cross the C-ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import _native as nat


def find_primes(bits: int, log_mod: int, count: int, exclude=()) -> list[int]:
    out = (C.c_uint64 * count)()
    ex = nat.u64_array(exclude)
    nat.call("lb_find_primes", bits, log_mod, count, ex, len(tuple(exclude)), out)
    return [int(v) for v in out]


@dataclass
class Params:
    """BFV-RNS parameter set. q: ciphertext primes, p: special primes,
    t: plaintext CRT primes (one independent BFV instance each)."""

    n: int
    q: list[int]
    p: list[int] = field(default_factory=list)
    t: list[int] = field(default_factory=list)
    dnum: int = 0
    seed: int = 0
    b: list[int] = field(default_factory=list)


def _stream_ptr(stream) -> int | None:
    """cudaStream_t of a torch stream (default: torch's current stream)."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream()
    return int(getattr(stream, "cuda_stream", stream)) or None


def _current_device() -> int:
    """torch's current CUDA device (the library's runtime is told explicitly)."""
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except Exception:
        return 0


class Context:
    """params: any object with n, q, p, b, t, dnum, seed (Params or
    params.BfvParams)."""

    def __init__(self, params):
        self.params = params
        b = list(getattr(params, "b", []))
        self._q = nat.u64_array(params.q)
        self._p = nat.u64_array(params.p)
        self._b = nat.u64_array(b)
        self._t = nat.u64_array(params.t)
        prm = nat.lb_params(params.n, len(params.q), len(params.p), len(b), len(params.t),
                            C.cast(self._q, nat.P64), C.cast(self._p, nat.P64), C.cast(self._b, nat.P64),
                            C.cast(self._t, nat.P64), params.dnum, params.seed, _current_device())
        h = C.c_void_p()
        nat.call("lb_context_create", C.byref(prm), C.byref(h))
        self.handle = h

    def close(self) -> None:
        if self.handle:
            nat.call("lb_context_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return self.params.n

    @property
    def primes(self) -> list[int]:
        return [*self.params.q, *self.params.p, *getattr(self.params, "b", []), *self.params.t]

    def prime_and_psi(self, index: int) -> tuple[int, int]:
        q, psi = C.c_uint64(), C.c_uint64()
        nat.call("lb_context_prime", self.handle, index, C.byref(q), C.byref(psi))
        return q.value, psi.value

    def sync(self, stream=None) -> None:
        nat.call("lb_sync", self.handle, _stream_ptr(stream))

    def _ntt(self, name, data, limbs, first_prime, polys, poly_stride, stream):
        import torch

        if not data.is_cuda or not data.is_contiguous():
            raise ValueError("NTT operand must be a contiguous CUDA tensor")
        if data.dtype == torch.int32:
            name += "_u32"  # u32 residue words (primes < 2^30)
        elif data.dtype != torch.int64:
            raise ValueError("NTT operand must be int64 (u64 residues) or int32 (u32 residues)")
        n = self.n
        if polys is None:
            polys = data.numel() // (limbs * n)
        if poly_stride is None:
            poly_stride = limbs * n
        if (polys - 1) * poly_stride + limbs * n > data.numel():
            raise ValueError("tensor too small for the described batch")
        nat.call(name, self.handle, data.data_ptr(), polys, limbs, first_prime, poly_stride, _stream_ptr(stream))

    def ntt_forward(self, data, limbs: int, first_prime: int = 0, polys=None, poly_stride=None, stream=None):
        """In place; data is [polys][limbs][n] int64 (u64 residues) or int32
        (u32 residues, primes < 2^30) on the device."""
        self._ntt("lb_ntt_forward", data, limbs, first_prime, polys, poly_stride, stream)

    def ntt_inverse(self, data, limbs: int, first_prime: int = 0, polys=None, poly_stride=None, stream=None):
        self._ntt("lb_ntt_inverse", data, limbs, first_prime, polys, poly_stride, stream)


def bitrev_perm(n: int):
    """perm[k] = bitrev(k) over log2(n) bits, as a numpy array."""
    import numpy as np

    bits = n.bit_length() - 1
    k = np.arange(n, dtype=np.int64)
    r = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        r |= ((k >> b) & 1) << (bits - 1 - b)
    return r
