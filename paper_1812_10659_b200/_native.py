"""ctypes binding of the C-ABI in include/lola_b200.h.

The shared library is built in-tree by build.py. There is no fallback: if the
library is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "liblola_b200.so"
if os.environ.get("LB_LIB"):  # experiment builds (build.py LB_VARIANT)
    LIB_PATH = Path(__file__).resolve().parent / "lib" / "variants" / os.environ["LB_LIB"] / "liblola_b200.so"

u32, u64, i32, i64, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_void_p
P64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)


class LolaError(RuntimeError):
    """Nonzero status from the C-ABI (1 internal / CUDA)."""

    code = 1


class BudgetError(LolaError):
    """Status 4: depth or magnitude budget exhausted (depth_error / magnitude_error)."""

    code = 4


class lb_params(C.Structure):
    _fields_ = [("n", u32), ("num_q", u32), ("num_p", u32), ("num_b", u32), ("num_t", u32),
                ("q", P64), ("p", P64), ("b", P64), ("t", P64), ("dnum", u32), ("seed", u64), ("device", i32)]


# name -> argtypes; every function returns int status except lb_last_error.
_SIGS: dict[str, list] = {
    "lb_find_primes": [u32, u32, u32, P64, u32, P64],
    "lb_context_create": [C.POINTER(lb_params), C.POINTER(vp)],
    "lb_context_destroy": [vp],
    "lb_context_prime": [vp, u32, P64, P64],
    "lb_context_residue_bytes": [vp, C.POINTER(u32)],
    "lb_pool_reserve": [vp, u64],
    "lb_sync": [vp, vp],
    "lb_ntt_forward": [vp, vp, u32, u32, u32, u64, vp],
    "lb_ntt_inverse": [vp, vp, u32, u32, u32, u64, vp],
    "lb_ntt_forward_u32": [vp, vp, u32, u32, u32, u64, vp],
    "lb_ntt_inverse_u32": [vp, vp, u32, u32, u32, u64, vp],
    "lb_bench_butterfly_peak": [u64, C.c_int, C.c_int, C.POINTER(C.c_double)],
    "lb_bench_int_pipes": [C.c_int, C.POINTER(C.c_double)],
    "lb_encrypt_slots": [vp, vp, u32, u64, vp, vp],
    "lb_decrypt_slots": [vp, vp, u32, vp, vp],
    "lb_decrypt_coeffs": [vp, vp, u32, vp, vp],
    "lb_encode_plain": [vp, vp, vp, vp, vp],
    "lb_ct_add": [vp, vp, vp, vp, u32, vp],
    "lb_ct_mul_scalar": [vp, vp, i64, vp, u32, vp],
    "lb_ct_mul_plain": [vp, vp, vp, vp, u32, vp],
    "lb_ct_add_plain": [vp, vp, vp, vp, u32, vp],
    "lb_ct_rotate": [vp, vp, u64, vp, u32, vp],
    "lb_ct_mul": [vp, vp, vp, vp, u32, vp],
    "lb_keygen": [vp, u64, vp],
    "lb_key_pointer": [vp, u64, C.POINTER(vp)],
    "lb_automorphism": [vp, vp, vp, u32, u32, u64, vp],
    "lb_key_switch": [vp, vp, u64, vp, vp, u32, vp],
}

# functions returning a value rather than a status
_VALUE_SIGS: dict[str, tuple] = {
    "lb_galois_exponent_columns": (u64, [u32, u32]),
    "lb_galois_exponent_rows": (u64, [u32]),
    "lb_launch_count": (u64, []),
}

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise LolaError(f"native library not built: {LIB_PATH} (run paper_1812_10659_b200/build.py)")
        l = C.CDLL(str(LIB_PATH))
        l.lb_last_error.restype = C.c_char_p
        l.lb_last_error.argtypes = []
        for name, args in _SIGS.items():
            fn = getattr(l, name)
            fn.argtypes = args
            fn.restype = C.c_int
        for name, (res, args) in _VALUE_SIGS.items():
            fn = getattr(l, name)
            fn.argtypes = args
            fn.restype = res
        _lib = l
    return _lib


def register(sigs: dict) -> None:
    """Add status-returning signatures (used by modules defining structs)."""
    _SIGS.update(sigs)
    if _lib is not None:
        for name, args in sigs.items():
            fn = getattr(_lib, name)
            fn.argtypes = args
            fn.restype = C.c_int


def declared_symbols() -> list[str]:
    return ["lb_last_error", *_SIGS, *_VALUE_SIGS]


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().lb_last_error().decode(errors="replace")
    if status == 3:
        raise ValueError(msg)
    if status == 4:
        raise BudgetError(msg)
    raise LolaError(f"status {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def u64_array(values) -> C.Array:
    vals = [int(v) for v in values]
    return (C.c_uint64 * max(1, len(vals)))(*vals)
