"""ctypes binding of oracle/_ref/libpackref.so — the UNMODIFIED reference
(packnn) compiled in place with the Boost stand-in and the shim in
oracle/ref_shim.cpp.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs as the checker or the CPU
baseline, never by the product package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libpackref.so"

u32, u64, i32, i64, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_void_p
P64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)
PF64 = C.POINTER(C.c_double)
PU32 = C.POINTER(C.c_uint32)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"reference status {code}: {msg}")
        self.code = code


class pref_stage(C.Structure):
    _fields_ = [("is_conv", i32), ("maps", u32), ("win_h", u32), ("win_w", u32), ("stride_h", u32),
                ("stride_w", u32), ("pad_top", u32), ("pad_left", u32), ("pad_bottom", u32),
                ("pad_right", u32), ("cols", u64), ("weights", PI64), ("bias", PI64)]


class pref_net(C.Structure):
    _fields_ = [("channels", u32), ("in_h", u32), ("in_w", u32), ("num_stages", u32),
                ("stages", C.POINTER(pref_stage)), ("input_bound", i64)]


_SIGS = {
    "pref_find_root_of_unity": [u64, u64, P64],
    "pref_ntt_forward": [u64, u32, P64, P64],
    "pref_ntt_inverse": [u64, u32, P64, P64],
    "pref_ntt_forward_many": [u64, u32, u64, P64, P64, C.c_int, PF64],
    "pref_slot_to_eval": [u64, u32, PU32],
    "pref_poly_mul": [u64, u32, P64, P64, P64],
    "pref_poly_add": [u64, u32, P64, P64, P64],
    "pref_poly_scale": [u64, u32, P64, u64, P64],
    "pref_slot_encode": [u64, u32, P64, P64],
    "pref_slot_decode": [u64, u32, P64, P64],
    "pref_galois_apply": [u64, u32, P64, u64, P64],
    "pref_galois_exponent_columns": [u32, u32, P64],
    "pref_crt_join_center": [P64, P64, u32, C.c_int, C.c_char_p, u64],
    "pref_schoolbook_mul": [u64, u32, P64, P64, P64],
    "pref_eval_rotate": [u64, u32, C.c_int, PI64, i64, C.c_int, PI64],
    "pref_forward_integer": [C.POINTER(pref_net), PI64, C.c_char_p, u64],
    "pref_final_bound": [C.POINTER(pref_net), C.c_char_p, u64],
    "pref_render_trace": [C.POINTER(pref_net), C.c_char_p, u32, P64, u32, C.c_char_p, u64],
    "pref_run_plan": [C.POINTER(pref_net), C.c_char_p, u32, P64, u32, C.c_int, u32, PI64, C.c_char_p, u64,
                      P64, u32, PU32, PF64],
    "pref_time_plan_steps": [C.POINTER(pref_net), C.c_char_p, u32, P64, u32, C.c_int, u32, PI64, PF64, u32,
                             PU32, PF64],
    "pref_time_primitives": [u64, u32, u32, PF64],
    "pref_session_create": [C.POINTER(pref_net), C.c_char_p, u32, P64, u32, C.c_int, u32, C.POINTER(vp)],
    "pref_session_destroy": [vp],
    "pref_session_run": [vp, PI64, C.c_int, C.c_char_p, u64, PF64],
}

_lib = None
# the drop-in proof: the reference's unmodified plan/kernels/representations
# over the B200 evaluator (oracle/b200_dropin/evaluator_b200.cpp)
DROPIN_LIB = HERE / "_ref" / "libpackb200.so"
_dropin = None


def available() -> bool:
    return REF_LIB.exists()


def _load(path: Path):
    if not path.exists():
        raise RefError(-1, f"{path} not built (make -C oracle)")
    l = C.CDLL(str(path))
    l.pref_last_error.restype = C.c_char_p
    l.pref_galois_exponent_rows.restype = u64
    l.pref_galois_exponent_rows.argtypes = [u32]
    l.pref_is_prime.argtypes = [u64]
    for name, args in _SIGS.items():
        f = getattr(l, name)
        f.argtypes = args
        f.restype = C.c_int
    return l


def lib():
    global _lib
    if _lib is None:
        _lib = _load(REF_LIB)
    return _lib


def dropin_lib():
    global _dropin
    if _dropin is None:
        l = _load(DROPIN_LIB)
        l.pb2_set_params.argtypes = [P64, u32, P64, u32, P64, u32, u32, u64]
        l.pb2_set_params.restype = C.c_int
        _dropin = l
    return _dropin


def run_plan_b200(net, strategy: str, prm, x):
    """The reference's own plan (build_plan + encode_input + execute +
    decode, proj/src/plan.cpp:582-633) on the B200 evaluator backend
    (BackendKind 2) with BFV parameters `prm`. Returns (scores, per-step
    counters)."""
    l = dropin_lib()
    q, pp, b = _arr(prm.q), _arr(prm.p), _arr(prm.b)
    l.pb2_set_params(_u64(q), q.size, _u64(pp), pp.size, _u64(b), b.size, prm.dnum, prm.seed)
    h = NetHandle(net)
    t = _arr(prm.t)
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    buf = C.create_string_buffer(1 << 22)
    counters = np.zeros(7 * 64, dtype=np.uint64)
    steps = C.c_uint32()
    times = np.zeros(3, dtype=np.float64)
    rc = l.pref_run_plan(h.ptr(), strategy.encode(), prm.n, _u64(t), t.size, 2, 1, xv.ctypes.data_as(PI64), buf,
                         1 << 22, _u64(counters), 64, C.byref(steps), times.ctypes.data_as(PF64))
    if rc:
        raise RefError(rc, l.pref_last_error().decode())
    scores = [int(v) for v in buf.value.decode().split(",")]
    return scores, counters[: 7 * steps.value].reshape(-1, 7).astype(np.int64)


def _check(rc: int) -> None:
    if rc:
        raise RefError(rc, lib().pref_last_error().decode())


def _u64(a: np.ndarray):
    return a.ctypes.data_as(P64)


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def root_of_unity(p: int, order: int) -> int:
    out = C.c_uint64()
    _check(lib().pref_find_root_of_unity(p, order, C.byref(out)))
    return out.value


def is_prime(v: int) -> bool:
    return bool(lib().pref_is_prime(v))


def ntt_forward(p: int, coeffs) -> np.ndarray:
    a = _arr(coeffs)
    out = np.empty_like(a)
    _check(lib().pref_ntt_forward(p, a.size, _u64(a), _u64(out)))
    return out


def ntt_inverse(p: int, evals) -> np.ndarray:
    a = _arr(evals)
    out = np.empty_like(a)
    _check(lib().pref_ntt_inverse(p, a.size, _u64(a), _u64(out)))
    return out


def ntt_many_seconds(p: int, n: int, limbs: np.ndarray, inverse: bool = False) -> tuple[np.ndarray, float]:
    a = _arr(limbs).reshape(-1)
    out = np.empty_like(a)
    sec = C.c_double()
    _check(lib().pref_ntt_forward_many(p, n, a.size // n, _u64(a), _u64(out), int(inverse), C.byref(sec)))
    return out.reshape(-1, n), sec.value


def time_primitives(p: int, n: int, reps: int = 5) -> dict:
    """Seconds per limb of the reference's forward / inverse NTT,
    poly_mul_negacyclic and galois_apply (tables built once)."""
    out = np.zeros(4, dtype=np.float64)
    _check(lib().pref_time_primitives(p, n, reps, out.ctypes.data_as(PF64)))
    return dict(zip(("ntt_forward", "ntt_inverse", "poly_mul", "galois_apply"), out.tolist()))


def slot_to_eval(p: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    _check(lib().pref_slot_to_eval(p, n, out.ctypes.data_as(PU32)))
    return out


def _binary(name: str, p: int, a, b) -> np.ndarray:
    a, b = _arr(a), _arr(b)
    out = np.empty_like(a)
    _check(getattr(lib(), name)(p, a.size, _u64(a), _u64(b), _u64(out)))
    return out


def poly_mul(p, a, b):
    return _binary("pref_poly_mul", p, a, b)


def poly_add(p, a, b):
    return _binary("pref_poly_add", p, a, b)


def schoolbook_mul(p, a, b):
    return _binary("pref_schoolbook_mul", p, a, b)


def poly_scale(p: int, a, s: int) -> np.ndarray:
    a = _arr(a)
    out = np.empty_like(a)
    _check(lib().pref_poly_scale(p, a.size, _u64(a), s, _u64(out)))
    return out


def slot_encode(p: int, slots) -> np.ndarray:
    a = _arr(slots)
    out = np.empty_like(a)
    _check(lib().pref_slot_encode(p, a.size, _u64(a), _u64(out)))
    return out


def slot_decode(p: int, coeffs) -> np.ndarray:
    a = _arr(coeffs)
    out = np.empty_like(a)
    _check(lib().pref_slot_decode(p, a.size, _u64(a), _u64(out)))
    return out


def galois_apply(p: int, coeffs, exponent: int) -> np.ndarray:
    a = _arr(coeffs)
    out = np.empty_like(a)
    _check(lib().pref_galois_apply(p, a.size, _u64(a), exponent, _u64(out)))
    return out


def galois_exponent_columns(n: int, k: int) -> int:
    out = C.c_uint64()
    _check(lib().pref_galois_exponent_columns(n, k, C.byref(out)))
    return out.value


def galois_exponent_rows(n: int) -> int:
    return int(lib().pref_galois_exponent_rows(n))


def crt_join_center(residues, primes, center: bool = True) -> int:
    r, p = _arr(residues), _arr(primes)
    buf = C.create_string_buffer(256)
    _check(lib().pref_crt_join_center(_u64(r), _u64(p), r.size, int(center), buf, 256))
    return int(buf.value.decode())


def eval_rotate(p: int, n: int, values, k: int, rows: bool, ring: bool) -> np.ndarray:
    v = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    out = np.empty(n, dtype=np.int64)
    _check(lib().pref_eval_rotate(p, n, int(ring), v.ctypes.data_as(PI64), k, int(rows), out.ctypes.data_as(PI64)))
    return out


# ---- networks ---------------------------------------------------------------

class NetHandle:
    """Keeps the ctypes structures (and the numpy arrays they point into) alive."""

    def __init__(self, net):
        self.keep = []
        stages = (pref_stage * len(net.stages))()
        for i, st in enumerate(net.stages):
            w = np.ascontiguousarray(st.weights, dtype=np.int64).reshape(-1)
            b = None if st.bias is None else np.ascontiguousarray(st.bias, dtype=np.int64)
            self.keep += [w, b]
            s = stages[i]
            s.is_conv = 1 if st.is_conv else 0
            s.maps = st.rows
            s.win_h, s.win_w = st.win
            s.stride_h, s.stride_w = st.stride
            s.pad_top, s.pad_left, s.pad_bottom, s.pad_right = st.pad
            s.cols = st.cols
            s.weights = w.ctypes.data_as(PI64)
            s.bias = b.ctypes.data_as(PI64) if b is not None else C.cast(None, PI64)
        self.keep.append(stages)
        c, h, w_ = net.input_shape
        self.net = pref_net(c, h, w_, len(net.stages), stages, net.input_bound)

    def ptr(self):
        return C.byref(self.net)


def forward_integer(net, x) -> list[int]:
    h = NetHandle(net)
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    buf = C.create_string_buffer(1 << 20)
    _check(lib().pref_forward_integer(h.ptr(), xv.ctypes.data_as(PI64), buf, 1 << 20))
    return [int(s) for s in buf.value.decode().split(",")]


def final_bound(net) -> int:
    h = NetHandle(net)
    buf = C.create_string_buffer(4096)
    _check(lib().pref_final_bound(h.ptr(), buf, 4096))
    return int(buf.value.decode())


def render_trace(net, strategy: str, n: int, primes) -> str:
    h = NetHandle(net)
    p = _arr(primes)
    buf = C.create_string_buffer(1 << 16)
    _check(lib().pref_render_trace(h.ptr(), strategy.encode(), n, _u64(p), p.size, buf, 1 << 16))
    return buf.value.decode()


def run_plan(net, strategy: str, n: int, primes, x, ring: bool = True, threads: int = 1):
    """Reference plaintext-semantics inference. Returns (scores, per-step
    counters [steps x 7], times {encode, steps(+decode)})."""
    h = NetHandle(net)
    p = _arr(primes)
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    buf = C.create_string_buffer(1 << 22)
    counters = np.zeros(7 * 64, dtype=np.uint64)
    steps = C.c_uint32()
    times = np.zeros(3, dtype=np.float64)
    _check(lib().pref_run_plan(h.ptr(), strategy.encode(), n, _u64(p), p.size, int(ring), threads,
                               xv.ctypes.data_as(PI64), buf, 1 << 22, _u64(counters), 64, C.byref(steps),
                               times.ctypes.data_as(PF64)))
    scores = [int(s) for s in buf.value.decode().split(",")]
    return scores, counters[: 7 * steps.value].reshape(-1, 7).astype(np.int64), times


def time_plan_steps(net, strategy: str, n: int, primes, x, ring: bool = True, threads: int = 1):
    h = NetHandle(net)
    p = _arr(primes)
    xv = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
    st = np.zeros(64, dtype=np.float64)
    steps = C.c_uint32()
    enc = C.c_double()
    _check(lib().pref_time_plan_steps(h.ptr(), strategy.encode(), n, _u64(p), p.size, int(ring), threads,
                                      xv.ctypes.data_as(PI64), st.ctypes.data_as(PF64), 64, C.byref(steps),
                                      C.byref(enc)))
    return enc.value, st[: steps.value]


class RefSession:
    """Network, EvalContext and plan built once (pref_session_create); each
    run() is the reference's per-image work: encode_input + every plan step
    (+ decode when asked). Returns (scores or None, [encode, steps, decode] s)."""

    def __init__(self, net, strategy: str, n: int, primes, ring: bool = True, threads: int = 1):
        self._h = NetHandle(net)
        p = _arr(primes)
        h = vp()
        _check(lib().pref_session_create(self._h.ptr(), strategy.encode(), n, _u64(p), p.size, int(ring), threads,
                                         C.byref(h)))
        self.handle = h

    def run(self, x, decode: bool = False):
        xv = np.ascontiguousarray(np.asarray(x, dtype=np.int64))
        times = np.zeros(3, dtype=np.float64)
        cap = (1 << 22) if decode else 1
        buf = C.create_string_buffer(cap)
        _check(lib().pref_session_run(self.handle, xv.ctypes.data_as(PI64), int(decode), buf, cap,
                                      times.ctypes.data_as(PF64)))
        scores = [int(v) for v in buf.value.decode().split(",")] if decode else None
        return scores, times

    def close(self):
        if getattr(self, "handle", None):
            lib().pref_session_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
