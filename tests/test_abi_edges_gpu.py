"""C-ABI edge cases on the device: empty batches, invalid arguments (status 3
= std::invalid_argument, as the reference's CLI maps it), aliasing outputs,
and the residue word reported per context (u32 for primes below 2^30)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_1812_10659_b200 import _native as nat
from paper_1812_10659_b200.bfv import BfvContext, galois_exponent_columns
from paper_1812_10659_b200.params import make_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[60, 29], ids=["u64", "u32"])
def cx(request):
    return BfvContext(make_params(4096, L=4, T=2, K=2, dnum=2, bits=request.param, seed=5))


def test_residue_word_follows_the_primes(cx):
    rb = C.c_uint32()
    nat.call("lb_context_residue_bytes", cx.handle, C.byref(rb))
    small = max(cx.params.q + cx.params.p) < 2**30
    assert rb.value == (4 if small else 8)
    assert cx.res_dtype == (torch.int32 if small else torch.int64)
    ct = cx.encrypt_slots(torch.zeros((1, cx.n), dtype=torch.int64, device="cuda"))
    assert ct.dtype == cx.res_dtype and ct.shape == (1, cx.T, 2, cx.L, cx.n)


def test_empty_batches_are_no_ops(cx):
    a = cx.empty_cts(0)
    nat.call("lb_ct_add", cx.handle, a.data_ptr() or 1, a.data_ptr() or 1, a.data_ptr() or 1, 0, None)
    nat.call("lb_ct_rotate", cx.handle, a.data_ptr() or 1, galois_exponent_columns(cx.n, 1), a.data_ptr() or 1, 0, None)
    nat.call("lb_ct_mul", cx.handle, a.data_ptr() or 1, a.data_ptr() or 1, a.data_ptr() or 1, 0, None)
    out = torch.empty((0, cx.T, cx.n), dtype=torch.int64, device="cuda")
    nat.call("lb_decrypt_slots", cx.handle, a.data_ptr() or 1, 0, out.data_ptr() or 1, None)
    torch.cuda.synchronize()


def test_invalid_arguments_raise_status_3(cx):
    ct = cx.encrypt_slots(torch.ones((1, cx.n), dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="galois"):
        cx.rotate(ct, 4)  # even element
    with pytest.raises(ValueError, match="galois"):
        cx.rotate(ct, 2 * cx.n + 1)  # out of range
    with pytest.raises(ValueError, match="null"):
        nat.call("lb_ct_add", cx.handle, None, ct.data_ptr(), ct.data_ptr(), 1, None)
    with pytest.raises(ValueError):
        cx.add(ct.to(torch.float32), ct)  # wrong residue dtype is rejected before the ABI


def test_aliasing_outputs(cx):
    """out == input for add, scalar and rotation gives the same result as a
    fresh output (the rotation gathers its input through the automorphism)."""
    rng = np.random.default_rng(1)
    v = torch.from_numpy(rng.integers(-50, 50, size=(1, cx.n), dtype=np.int64)).cuda()
    ct = cx.encrypt_slots(v, id_base=3)
    g = galois_exponent_columns(cx.n, 3)
    want_rot = cx.rotate(ct, g)
    want_add = cx.add(ct, want_rot)
    x = ct.clone()
    cx.rotate(x, g, out=x)
    assert torch.equal(x, want_rot)
    cx.add(ct, x, out=x)
    assert torch.equal(x, want_add)
    want_sc = cx.mul_scalar(ct, -7)
    y = ct.clone()
    cx.mul_scalar(y, -7, out=y)
    assert torch.equal(y, want_sc)
    m = cx.decrypt_slots(want_add).cpu().numpy()
    vals = v.cpu().numpy()[0]
    half = cx.n // 2
    rot = np.concatenate([np.roll(vals[:half], 3), np.roll(vals[half:], 3)])
    for j, t in enumerate(cx.params.t):
        assert np.array_equal(m[0, j], np.mod(vals + rot, t))


def test_pool_reserve_then_ops(cx):
    """lb_pool_reserve grows the allocation pool up front; later ops reuse it."""
    free0, _ = torch.cuda.mem_get_info()
    nat.call("lb_pool_reserve", cx.handle, 1 << 28)
    ct = cx.encrypt_slots(torch.ones((1, cx.n), dtype=torch.int64, device="cuda"))
    out = cx.add(ct, ct)
    m = cx.decrypt_slots(out).cpu().numpy()
    assert (m[0] == 2).all()
    free1, _ = torch.cuda.mem_get_info()
    assert free1 <= free0  # the reserved memory stays with the pool
