"""The drop-in library (oracle/_ref/libpackb200.so: the reference's plan,
kernels and representations over the B200 evaluator) builds and loads
without a GPU, links this repo's liblola_b200.so, and carries only the b200
backend (the reference's Slot/Ring requests are refused)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import refbind as R
from paper_1812_10659_b200 import nets


def test_dropin_library_loads_and_refuses_other_backends():
    if not R.DROPIN_LIB.exists():
        pytest.skip("oracle/_ref/libpackb200.so not built")
    l = R.dropin_lib()
    assert l.pb2_available() == 1
    maps = open("/proc/self/maps").read()
    assert "liblola_b200" in maps
    net = nets.toy_net()
    h = R.NetHandle(net)
    t = np.array([2148728833, 2148794369, 2149810177], dtype=np.uint64)
    x = np.ascontiguousarray(nets.images(9, net, 1)[0])
    buf = C.create_string_buffer(4096)
    cnt = np.zeros(7 * 64, dtype=np.uint64)
    steps = C.c_uint32()
    times = np.zeros(3)
    rc = l.pref_run_plan(h.ptr(), b"lola-mnist", 4096, t.ctypes.data_as(R.P64), 3, 1, 1,
                         x.ctypes.data_as(R.PI64), buf, 4096, cnt.ctypes.data_as(R.P64), 64, C.byref(steps),
                         times.ctypes.data_as(R.PF64))
    assert rc == 3 and b"only the b200 backend" in l.pref_last_error()
