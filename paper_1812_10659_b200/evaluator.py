"""Python mirror of the reference's evaluator boundary over the C-ABI.

Same names, argument meaning and error behaviour as packnn's
EvalContext / Evaluator (proj/include/packnn/evaluator.hpp:16-91) and
Message (proj/include/packnn/message.hpp:66-75), on device BFV ciphertexts:

    reference                         here
    EvalContext(kind, n, primes, d)   EvalContext(bfv_context, batch, max_depth)
    Evaluator::lift / lower           Evaluator.lift / lower (batched)
    add, add_plain, mul, mul_plain,   same names
    mask, mul_scalar, rotate_columns,
    rotate_rows, rotate_bundle,
    fork, absorb
    depth_error / magnitude_error     DepthError / MagnitudeError
    std::invalid_argument             ValueError

A Message holds a batch of `batch` independent messages; lifted values are
shared by all of them unless given per message.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .lola import words_to_int

vp = C.c_void_p
P64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)

nat.register({
    "lb_eval_create": [vp, C.c_uint32, C.c_uint32, vp, C.POINTER(vp)],
    "lb_eval_destroy": [vp],
    "lb_eval_fork": [vp, C.POINTER(vp)],
    "lb_eval_absorb": [vp, vp],
    "lb_eval_counters": [vp, P64],
    "lb_eval_note_live": [vp, C.c_uint64],
    "lb_eval_lift": [vp, PI64, C.c_uint64, C.c_int, C.POINTER(vp)],
    "lb_eval_lower": [vp, vp, P64],
    "lb_eval_add": [vp, vp, vp, C.POINTER(vp)],
    "lb_eval_add_plain": [vp, vp, PI64, C.c_uint64, C.POINTER(vp)],
    "lb_eval_mul": [vp, vp, vp, C.POINTER(vp)],
    "lb_eval_mul_plain": [vp, vp, PI64, C.c_uint64, C.POINTER(vp)],
    "lb_eval_mask": [vp, vp, C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(vp)],
    "lb_eval_mul_scalar": [vp, vp, C.c_int64, C.POINTER(vp)],
    "lb_eval_rotate_columns": [vp, vp, C.c_int64, C.POINTER(vp)],
    "lb_eval_rotate_rows": [vp, vp, C.POINTER(vp)],
    "lb_eval_rotate_bundle": [vp, vp, C.c_uint32, C.POINTER(vp)],
    "lb_message_free": [vp],
    "lb_message_info": [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.c_char_p, C.c_uint64],
    "lb_message_data": [vp, C.POINTER(vp)],
})


class DepthError(nat.BudgetError):
    """depth_error (proj/include/packnn/message.hpp:14-18)."""


class MagnitudeError(nat.BudgetError):
    """magnitude_error (proj/include/packnn/message.hpp:20-24)."""


def _call(name, *args):
    try:
        nat.call(name, *args)
    except nat.BudgetError as e:
        msg = str(e)
        raise (MagnitudeError if "magnitude" in msg else DepthError)(msg) from None


class Message:
    """Opaque handle of one batched message (device ciphertexts)."""

    def __init__(self, handle):
        self.handle = handle

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                nat.call("lb_message_free", self.handle)
            except Exception:
                pass
            self.handle = None

    def _info(self):
        d, pd = C.c_uint32(), C.c_uint32()
        buf = C.create_string_buffer(128)
        nat.call("lb_message_info", self.handle, C.byref(d), C.byref(pd), buf, 128)
        return d.value, pd.value, int(buf.value.decode())

    @property
    def depth(self) -> int:
        return self._info()[0]

    @property
    def plain_depth(self) -> int:
        return self._info()[1]

    @property
    def magnitude(self) -> int:
        return self._info()[2]


class EvalContext:
    def __init__(self, bfv_context, batch: int = 1, max_depth: int = 8):
        self.device = bfv_context
        self.batch = batch
        self.max_depth = max_depth

    @property
    def n(self) -> int:
        return self.device.n

    @property
    def half(self) -> int:
        return self.device.n // 2


class Evaluator:
    def __init__(self, cx: EvalContext, _handle=None):
        self.cx = cx
        if _handle is None:
            h = vp()
            import torch

            s = torch.cuda.current_stream()
            nat.call("lb_eval_create", cx.device.handle, cx.batch, cx.max_depth, int(s.cuda_stream) or None,
                     C.byref(h))
            _handle = h
        self.handle = _handle

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                nat.call("lb_eval_destroy", self.handle)
            except Exception:
                pass
            self.handle = None

    def context(self) -> EvalContext:
        return self.cx

    # ---- counters ------------------------------------------------------------
    def counters(self) -> dict:
        out = (C.c_uint64 * 8)()
        nat.call("lb_eval_counters", self.handle, out)
        keys = ("ct_ct_mul", "ct_plain_mul", "scalar_mul", "mask_mul", "add", "rot_cols", "rot_rows",
                "live_messages_peak")
        return dict(zip(keys, (int(v) for v in out)))

    def note_live(self, live: int) -> None:
        nat.call("lb_eval_note_live", self.handle, live)

    def fork(self) -> "Evaluator":
        h = vp()
        nat.call("lb_eval_fork", self.handle, C.byref(h))
        return Evaluator(self.cx, _handle=h)

    def absorb(self, child: "Evaluator") -> None:
        nat.call("lb_eval_absorb", self.handle, child.handle)

    # ---- encoding boundary -------------------------------------------------------
    def lift(self, values, per_message: bool = False) -> Message:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
        count = v.shape[-1] if v.ndim else 0
        if per_message and v.shape[0] != self.cx.batch:
            raise ValueError("per-message values need one row per batch entry")
        h = vp()
        _call("lb_eval_lift", self.handle, v.ctypes.data_as(PI64), count, int(per_message), C.byref(h))
        return Message(h)

    def lower(self, m: Message):
        """[batch][n] Python ints (centered CRT of every slot)."""
        out = np.zeros((self.cx.batch, self.cx.n, 4), dtype=np.uint64)
        nat.call("lb_eval_lower", self.handle, m.handle, out.ctypes.data_as(P64))
        return [[words_to_int(out[b, i]) for i in range(self.cx.n)] for b in range(self.cx.batch)]

    # ---- counted operations --------------------------------------------------------
    def _op(self, name, *args) -> Message:
        h = vp()
        _call(name, self.handle, *args, C.byref(h))
        return Message(h)

    def add(self, a: Message, b: Message) -> Message:
        return self._op("lb_eval_add", a.handle, b.handle)

    def add_plain(self, a: Message, values) -> Message:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
        return self._op("lb_eval_add_plain", a.handle, v.ctypes.data_as(PI64), v.size)

    def mul(self, a: Message, b: Message) -> Message:
        return self._op("lb_eval_mul", a.handle, b.handle)

    def mul_plain(self, a: Message, values) -> Message:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
        return self._op("lb_eval_mul_plain", a.handle, v.ctypes.data_as(PI64), v.size)

    def mask(self, a: Message, bits) -> Message:
        v = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8))
        return self._op("lb_eval_mask", a.handle, v.ctypes.data_as(C.POINTER(C.c_uint8)), v.size)

    def mul_scalar(self, a: Message, s: int) -> Message:
        return self._op("lb_eval_mul_scalar", a.handle, int(s))

    def rotate_columns(self, a: Message, k: int) -> Message:
        return self._op("lb_eval_rotate_columns", a.handle, int(k))

    def rotate_rows(self, a: Message) -> Message:
        return self._op("lb_eval_rotate_rows", a.handle)

    def rotate_bundle(self, a: Message, amount: int) -> Message:
        return self._op("lb_eval_rotate_bundle", a.handle, int(amount))
