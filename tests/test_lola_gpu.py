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


@pytest.mark.parametrize("bits", [60, 30])
def test_toy_cryptonets_simd_n4096(bits):
    """Record tensors: 5 images packed into the slots of one message per
    feature (plan.cpp:464-502); counters == the reference run on one record,
    every record's logits == forward_integer."""
    prm = make_params(4096, L=7 if bits == 60 else 14, T=3, K=1 if bits == 60 else 2,
                      dnum=0 if bits == 60 else 7, bits=bits, seed=7)
    _check(prm, nets.toy_net(), "cryptonets-simd", batch=5, config=9)


def test_lola_small_config3():
    _check(lola_small_params(), nets.lola_small_net(), "lola-small", batch=2, config=3)


def test_lola_mnist_config0():
    _check(lola_mnist_params(), nets.lola_mnist_net(), "lola-mnist", batch=2, config=0)


def test_lola_small_config3_word32():
    from paper_1812_10659_b200.params import lola_small_params_w32

    _check(lola_small_params_w32(), nets.lola_small_net(), "lola-small", batch=2, config=3)


def test_lola_mnist_config0_word32():
    """The same network on 30-bit RNS primes (32-bit word kernels)."""
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    _check(lola_mnist_params_w32(), nets.lola_mnist_net(), "lola-mnist", batch=2, config=0)


@pytest.mark.parametrize("word", [64, 32])
def test_lola_cifar_config4_single_image(word):
    """BASELINE config 4 (83 + 163 maps, 57,252 rotations per instance, 6
    plaintext primes): decrypted logits == forward_integer; per-step counters
    == the plan's predictions (checked inside execute) whose totals equal the
    golden trace proj/tests/golden/lola_cifar.txt:10."""
    from paper_1812_10659_b200.lola import plan_counters
    from paper_1812_10659_b200.params import lola_cifar_params, lola_cifar_params_w32

    net = nets.lola_cifar_net()
    prm = lola_cifar_params() if word == 64 else lola_cifar_params_w32()
    cx = BfvContext(prm)
    sess = Session(cx, net, "lola-cifar", 1)
    img = nets.images(4, net, 1)
    scores, counters, _ = sess.run(img)
    predicted, _, _ = plan_counters(net, "lola-cifar", prm.n)
    assert np.array_equal(counters, predicted)
    assert counters.sum(0).tolist() == [2, 8160, 15936, 4075, 81265, 53177, 4075]
    assert scores[0] == R.forward_integer(net, img[0])


def test_lola_mnist_w32_bench_batch():
    """Exactly the benched configuration: lola-mnist w32 (29-bit set, u32
    residues), the config-2 network and images, batch 64 (320 ciphertexts per
    key-switch launch). Every decrypted logit == forward_integer; counters ==
    the reference's."""
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    _check(lola_mnist_params_w32(), nets.lola_mnist_net(config=2), "lola-mnist", batch=64, config=2)


@pytest.mark.parametrize("which", ["toy", "mnist_w32"])
def test_cuda_graph_replay_matches(which):
    """Graph mode (lb_lola_session_set_graph): the captured plan replayed for
    new images (encrypt copies them into the captured input buffers) gives
    the same logits and counters as the direct path and forward_integer."""
    from paper_1812_10659_b200.params import lola_mnist_params_w32

    if which == "toy":
        prm, net, cfg, B = make_params(4096, L=7, T=3, K=1, seed=5), nets.toy_net(), 9, 2
    else:
        prm, net, cfg, B = lola_mnist_params_w32(), nets.lola_mnist_net(config=2), 2, 1
    cx = BfvContext(prm)
    sess = Session(cx, net, "lola-mnist", B)
    sess.set_graph(True)
    for start in (0, 5, 11):
        imgs = nets.images(cfg, net, B, start=start)
        scores, counters, _ = sess.run(imgs)
        for b in range(B):
            assert scores[b] == R.forward_integer(net, imgs[b]), f"images from {start}, image {b}"
    predicted, _, _ = __import__("paper_1812_10659_b200.lola", fromlist=["plan_counters"]).plan_counters(
        net, "lola-mnist", prm.n)
    assert np.array_equal(counters, predicted)
    # separate phases: encrypt once, replay execute several times
    imgs = nets.images(cfg, net, B, start=20)
    sess.encrypt(imgs)
    for _ in range(3):
        sess.execute()
    assert sess.decrypt() == [R.forward_integer(net, x) for x in imgs]
    sess.set_graph(False)
    sess.encrypt(imgs)
    sess.execute()
    assert sess.decrypt() == [R.forward_integer(net, x) for x in imgs]
