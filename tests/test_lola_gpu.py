"""End-to-end encrypted LoLa inference on the B200 against the reference:
decrypted logits == forward_integer (proj/src/layers.cpp:560-594) == the
reference ring-backend plan run, and measured per-step counters == the
reference's (proj/src/plan.cpp:617-621)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import refbind as R
from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.bfv import BfvContext
from paper_1812_10659_b200.lola import Session
from paper_1812_10659_b200.params import lola_mnist_params, lola_small_params, make_params

pytestmark = pytest.mark.gpu


def _check(prm, net, strategy, batch, config):
    cx = BfvContext(prm)
    sess = Session(cx, net, strategy, batch)
    imgs = nets.images(config, net, batch)
    scores, counters, _ = sess.run(imgs)
    ref_scores, ref_counters, _ = R.run_plan(net, strategy, prm.n, prm.t, imgs[0], ring=False)
    assert np.array_equal(counters, ref_counters)
    for b in range(batch):
        assert scores[b] == R.forward_integer(net, imgs[b]), f"image {b}"
    assert scores[0] == ref_scores
    return sess


def test_toy_lola_mnist_n4096():
    prm = make_params(4096, L=7, T=3, K=1, seed=5)
    _check(prm, nets.toy_net(), "lola-mnist", batch=3, config=9)


def test_toy_lola_dense_mnist_n4096():
    prm = make_params(4096, L=7, T=3, K=1, seed=6)
    _check(prm, nets.toy_net(), "lola-dense-mnist", batch=2, config=9)


def test_lola_small_config3():
    _check(lola_small_params(), nets.lola_small_net(), "lola-small", batch=2, config=3)


def test_lola_mnist_config0():
    _check(lola_mnist_params(), nets.lola_mnist_net(), "lola-mnist", batch=2, config=0)
