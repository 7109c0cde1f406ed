"""Encryption randomness is never reused within a context:
ciphertext ids come from one counter per context shared by every evaluator,
fork and session; default seeds come from OS entropy; the evaluator's
argument checks raise std::invalid_argument (status 3) like the reference
(proj/src/evaluator.cpp:70, 289-332); and plaintext-prime sets whose product
reaches 2^255 are refused (the device CRT writes 256-bit two's complement)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from paper_1812_10659_b200 import _native as nat
from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.bfv import BfvContext
from paper_1812_10659_b200.evaluator import EvalContext, Evaluator
from paper_1812_10659_b200.lola import Session
from paper_1812_10659_b200.params import find_primes, make_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cx():
    return BfvContext(make_params(4096, L=5, T=2, K=1, seed=77))


def _c1(msg_ptr, cx):
    """c1 of the first ciphertext of a message [B][T][2][L][n]."""
    from paper_1812_10659_b200.bfv import _DevPtr

    shape = (1, cx.T, 2, cx.L, cx.n)
    t = torch.as_tensor(_DevPtr(msg_ptr, shape, "<i8" if cx.res_dtype == torch.int64 else "<i4"), device="cuda")
    return t[0, 0, 1].clone()


def test_fresh_ids_by_default(cx):
    v = torch.ones((1, cx.n), dtype=torch.int64, device="cuda")
    a, b = cx.encrypt_slots(v), cx.encrypt_slots(v)
    assert not torch.equal(a[:, :, 1], b[:, :, 1]), "two encryptions shared their uniform component"
    # explicit ids reproduce (the oracle-parity hook)
    assert torch.equal(cx.encrypt_slots(v, id_base=9), cx.encrypt_slots(v, id_base=9))


def test_evaluators_and_forks_share_the_counter(cx):
    e1 = Evaluator(EvalContext(cx))
    e2 = Evaluator(EvalContext(cx))
    f = e1.fork()
    vals = list(range(10))
    ptrs = []
    for ev in (e1, e2, f, e1):
        m = ev.lift(vals)
        p = C.c_void_p()
        nat.call("lb_message_data", m.handle, C.byref(p))
        ptrs.append(_c1(p.value, cx))
        del m
    for i in range(len(ptrs)):
        for j in range(i + 1, len(ptrs)):
            assert not torch.equal(ptrs[i], ptrs[j]), f"messages {i} and {j} share randomness"


def test_sessions_on_one_context_draw_distinct_randomness():
    cx = BfvContext(make_params(4096, L=7, T=3, K=1, seed=5))  # the toy net needs 3 plaintext primes
    net = nets.toy_net()
    img = nets.images(9, net, 1)
    s1, s2 = Session(cx, net, "lola-mnist", 1), Session(cx, net, "lola-mnist", 1)
    s1.encrypt(img)
    s2.encrypt(img)
    s1.execute()
    s2.execute()
    o1, o2 = s1.output_ciphertexts(0), s2.output_ciphertexts(0)
    assert not torch.equal(o1[:, :, 1], o2[:, :, 1])
    assert s1.decrypt() == s2.decrypt()


def test_evaluator_argument_checks(cx):
    ev = Evaluator(EvalContext(cx))
    with pytest.raises(ValueError):
        ev.lift(list(range(cx.n + 1)))  # more values than slots
    m = ev.lift([1, 2, 3])
    with pytest.raises(ValueError):
        ev.rotate_columns(m, cx.n // 2)  # |k| < n/2
    with pytest.raises(ValueError):
        ev.rotate_bundle(m, cx.n // 2)
    with pytest.raises(ValueError):
        ev.mask(m, [0] * cx.n)  # empty mask
    with pytest.raises(ValueError):
        ev.mask(m, [2] + [0] * (cx.n - 1))  # entries must be 0 or 1


def test_plaintext_prime_product_capacity():
    """Five 62-bit plaintext primes (product ~2^310) pass the context's
    checks but not the evaluator's 2^255 CRT bound."""
    big_t = find_primes(62, 13, 5)
    prm = make_params(4096, L=5, T=5, K=1, seed=3, plain=big_t)
    cx = BfvContext(prm)
    with pytest.raises(ValueError, match="2\\^255"):
        Evaluator(EvalContext(cx))
