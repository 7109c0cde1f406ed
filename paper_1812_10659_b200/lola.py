"""LoLa encrypted inference over the C-ABI (include/lola_b200.h, §LoLa).

Mirrors the reference's plan interface (proj/include/packnn/plan.hpp:84-104):
`plan_counters` is build_plan's predicted step table, `Session.run` is
plan.encode_input -> execute -> decode with every counted operation a batched
BFV kernel sequence on the B200.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .nets import Network

u32, u64, i32, i64, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_void_p
PI64 = C.POINTER(C.c_int64)

COUNTER_NAMES = ("ct.ct", "ct.pt", "scalar", "mask", "add", "rot.col", "rot.row")


class lb_stage(C.Structure):
    _fields_ = [("is_conv", i32), ("maps", u32), ("win_h", u32), ("win_w", u32), ("stride_h", u32),
                ("stride_w", u32), ("pad_top", u32), ("pad_left", u32), ("pad_bottom", u32), ("pad_right", u32),
                ("cols", u64), ("weights", PI64), ("bias", PI64)]


class lb_network(C.Structure):
    _fields_ = [("channels", u32), ("in_h", u32), ("in_w", u32), ("num_stages", u32),
                ("stages", C.POINTER(lb_stage)), ("input_bound", i64)]


class lb_plan_options(C.Structure):
    """PlanOptions (proj/include/packnn/plan.hpp:35-41) minus the degree,
    which is the context's."""
    _fields_ = [("window_matrix_threshold", u64)]


DEFAULT_WINDOW_MATRIX_THRESHOLD = 100000


def _options(window_matrix_threshold: int):
    return C.byref(lb_plan_options(window_matrix_threshold))


_SIGS = {
    "lb_plan_counters": [C.POINTER(lb_network), C.c_char_p, u32, C.POINTER(C.c_uint64), u32,
                         C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)],
    "lb_plan_counters_ex": [C.POINTER(lb_network), C.c_char_p, u32, C.POINTER(lb_plan_options),
                            C.POINTER(C.c_uint64), u32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                            C.POINTER(C.c_uint64)],
    "lb_lola_session_create": [vp, C.POINTER(lb_network), C.c_char_p, u32, u32, vp, C.POINTER(vp)],
    "lb_lola_session_create_ex": [vp, C.POINTER(lb_network), C.c_char_p, u32, u32, C.POINTER(lb_plan_options), vp,
                                  C.POINTER(vp)],
    "lb_lola_session_destroy": [vp],
    "lb_lola_session_info": [vp, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "lb_lola_session_run": [vp, vp, C.c_int, vp, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_double)],
    "lb_lola_session_encrypt": [vp, vp, C.c_int],
    "lb_lola_session_execute": [vp, C.POINTER(C.c_uint64)],
    "lb_lola_session_decrypt": [vp, vp, C.c_int],
    "lb_lola_session_set_graph": [vp, C.c_int],
    "lb_lola_session_output": [vp, C.c_uint32, C.POINTER(vp), C.POINTER(C.c_uint32)],
}
nat.register(_SIGS)


class NetStruct:
    """ctypes view of a Network (keeps the numpy buffers alive)."""

    def __init__(self, net: Network):
        self.keep = []
        st = (lb_stage * len(net.stages))()
        for i, s in enumerate(net.stages):
            w = np.ascontiguousarray(s.weights, dtype=np.int64).reshape(-1)
            b = None if s.bias is None else np.ascontiguousarray(s.bias, dtype=np.int64)
            self.keep += [w, b]
            x = st[i]
            x.is_conv = 1 if s.is_conv else 0
            x.maps = s.rows
            x.win_h, x.win_w = s.win
            x.stride_h, x.stride_w = s.stride
            x.pad_top, x.pad_left, x.pad_bottom, x.pad_right = s.pad
            x.cols = s.cols
            x.weights = w.ctypes.data_as(PI64)
            x.bias = b.ctypes.data_as(PI64) if b is not None else C.cast(None, PI64)
        self.keep.append(st)
        c, h, w_ = net.input_shape
        self.s = lb_network(c, h, w_, len(net.stages), st, net.input_bound)

    def ptr(self):
        return C.byref(self.s)


def plan_counters(net: Network, strategy: str, n: int,
                  window_matrix_threshold: int = DEFAULT_WINDOW_MATRIX_THRESHOLD):
    """Predicted per-step counters [steps][7], depth needed, predicted peak."""
    ns = NetStruct(net)
    buf = (C.c_uint64 * (7 * 64))()
    steps, depth, peak = C.c_uint32(), C.c_uint32(), C.c_uint64()
    nat.call("lb_plan_counters_ex", ns.ptr(), strategy.encode(), n, _options(window_matrix_threshold), buf, 64,
             C.byref(steps), C.byref(depth), C.byref(peak))
    arr = np.frombuffer(buf, dtype=np.uint64)[: 7 * steps.value].reshape(-1, 7).astype(np.int64)
    return arr, depth.value, peak.value


def words_to_int(w) -> int:
    """Four little-endian u64 words, two's complement -> Python int."""
    v = int(w[0]) | int(w[1]) << 64 | int(w[2]) << 128 | int(w[3]) << 192
    return v - (1 << 256) if v >> 255 else v


class Session:
    """A plan bound to a BfvContext and a fixed batch of images."""

    def __init__(self, cx, net: Network, strategy: str, batch: int, max_depth: int = 8, stream=None,
                 window_matrix_threshold: int = DEFAULT_WINDOW_MATRIX_THRESHOLD):
        import torch

        self.cx, self.net, self.strategy, self.batch = cx, net, strategy, batch
        self._ns = NetStruct(net)
        s = torch.cuda.current_stream() if stream is None else stream
        self.stream = s
        h = vp()
        nat.call("lb_lola_session_create_ex", cx.handle, self._ns.ptr(), strategy.encode(), batch, max_depth,
                 _options(window_matrix_threshold), int(s.cuda_stream) or None, C.byref(h))
        self.handle = h
        steps, outs, ins = C.c_uint32(), C.c_uint64(), C.c_uint64()
        nat.call("lb_lola_session_info", h, C.byref(steps), C.byref(outs), C.byref(ins))
        self.steps, self.outputs, self.input_values = steps.value, outs.value, ins.value

    def set_graph(self, enable: bool = True) -> None:
        """CUDA-graph mode: execute captures the plan once and replays it."""
        nat.call("lb_lola_session_set_graph", self.handle, int(enable))

    def close(self):
        if getattr(self, "handle", None):
            nat.call("lb_lola_session_destroy", self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run_raw(self, images, scores, images_on_device: bool, scores_on_device: bool, want_counters=True,
                want_times=True):
        """images/scores: torch tensors (device) or numpy arrays (host)."""
        iptr = images.data_ptr() if images_on_device else images.ctypes.data
        sptr = scores.data_ptr() if scores_on_device else scores.ctypes.data
        counters = (C.c_uint64 * (7 * self.steps))() if want_counters else None
        times = (C.c_double * 3)() if want_times else None
        nat.call("lb_lola_session_run", self.handle, iptr, int(images_on_device), sptr, int(scores_on_device),
                 counters, times)
        cnt = np.frombuffer(counters, dtype=np.uint64).reshape(-1, 7).astype(np.int64) if want_counters else None
        return cnt, (list(times) if want_times else None)

    # separate phases (inputs resident on the device between them)
    def encrypt(self, images, on_device: bool = False) -> None:
        ptr = images.data_ptr() if on_device else np.ascontiguousarray(images, dtype=np.int64).ctypes.data
        if not on_device:
            self._host_images = images  # keep alive until the copy is issued
        nat.call("lb_lola_session_encrypt", self.handle, ptr, int(on_device))

    def execute(self, want_counters: bool = False):
        counters = (C.c_uint64 * (7 * self.steps))() if want_counters else None
        nat.call("lb_lola_session_execute", self.handle, counters)
        return np.frombuffer(counters, dtype=np.uint64).reshape(-1, 7).astype(np.int64) if want_counters else None

    def decrypt(self):
        scores = np.zeros((self.batch, self.outputs, 4), dtype=np.uint64)
        nat.call("lb_lola_session_decrypt", self.handle, scores.ctypes.data, 0)
        return [[words_to_int(scores[b, i]) for i in range(self.outputs)] for b in range(self.batch)]

    def output_ciphertexts(self, index: int):
        """Copy of encrypted output message `index`: torch [batch][T][2][L][n]."""
        import torch

        from .bfv import _DevPtr

        p, cnt = vp(), C.c_uint32()
        nat.call("lb_lola_session_output", self.handle, index, C.byref(p), C.byref(cnt))
        shape = (self.batch, len(self.cx.params.t), 2, len(self.cx.params.q), self.cx.n)
        typestr = "<i4" if self.cx.res_dtype == torch.int32 else "<i8"
        return torch.as_tensor(_DevPtr(p.value, shape, typestr), device="cuda").clone()

    def run(self, images: np.ndarray):
        """Host images [batch][input_values] -> (scores [batch][outputs] Python
        ints, per-step counters [steps][7], times (encode, steps, decode))."""
        images = np.ascontiguousarray(images, dtype=np.int64).reshape(self.batch, self.input_values)
        scores = np.zeros((self.batch, self.outputs, 4), dtype=np.uint64)
        cnt, times = self.run_raw(images, scores, False, False)
        out = [[words_to_int(scores[b, i]) for i in range(self.outputs)] for b in range(self.batch)]
        return out, cnt, times
