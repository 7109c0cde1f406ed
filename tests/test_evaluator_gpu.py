"""The evaluator boundary on device ciphertexts behaves like the reference's
Evaluator (cases follow proj/tests/test_backend.cpp:62-260 and
proj/tests/test_ring.cpp:126-141): values, magnitudes, depths, counters and
budget errors."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import refbind as R
from paper_1812_10659_b200.bfv import BfvContext
from paper_1812_10659_b200.evaluator import DepthError, EvalContext, Evaluator, MagnitudeError
from paper_1812_10659_b200.params import make_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    return BfvContext(make_params(4096, L=5, T=2, K=1, seed=21))


def test_add_sums_values_and_magnitudes(dev):
    ev = Evaluator(EvalContext(dev))
    r = ev.add(ev.lift([1, -2, 3]), ev.lift([10, 20, -30]))
    assert r.magnitude == 33
    assert ev.lower(r)[0][:3] == [11, 18, -27]
    assert ev.counters()["add"] == 1


def test_mul_consumes_depth_and_multiplies_magnitudes(dev):
    ev = Evaluator(EvalContext(dev, max_depth=2))
    m = ev.lift([3, -4])
    sq = ev.mul(m, m)
    assert sq.depth == 1 and sq.magnitude == 16
    assert ev.lower(sq)[0][:2] == [9, 16]
    sq2 = ev.mul(sq, sq)
    assert sq2.depth == 2 and ev.lower(sq2)[0][:2] == [81, 256]
    with pytest.raises(DepthError):
        ev.mul(sq2, sq2)
    assert ev.counters()["ct_ct_mul"] == 2


def test_magnitude_overflow_is_distinct_from_depth():
    cx = BfvContext(make_params(4096, L=3, T=1, K=1, seed=2))
    ev = Evaluator(EvalContext(cx, max_depth=10))
    m = ev.lift([1 << 16])
    with pytest.raises(MagnitudeError):
        ev.mul(m, m)  # 2^32 > (t - 1) / 2


def test_mul_plain_tracks_plain_depth(dev):
    ev = Evaluator(EvalContext(dev))
    r = ev.mul_plain(ev.lift([2, 3, -1]), [5, -6, 7])
    assert (r.plain_depth, r.depth, r.magnitude) == (1, 0, 21)
    assert ev.lower(r)[0][:3] == [10, -18, -7]
    assert ev.counters()["ct_plain_mul"] == 1


def test_scalar_and_add_plain(dev):
    ev = Evaluator(EvalContext(dev))
    m = ev.lift([5, -7, 9])
    s = ev.mul_scalar(m, -3)
    assert s.magnitude == 27 and s.plain_depth == 1
    assert ev.lower(s)[0][:3] == [-15, 21, -27]
    a = ev.add_plain(m, [1, 1, -10])
    assert ev.lower(a)[0][:3] == [6, -6, -1]
    c = ev.counters()
    assert (c["scalar_mul"], c["add"]) == (1, 1)


def test_rotations_follow_the_slot_matrix(dev):
    n, half = dev.n, dev.n // 2
    ev = Evaluator(EvalContext(dev))
    vals = np.arange(n, dtype=np.int64) - half
    m = ev.lift(vals)
    row0, row1 = vals[:half], vals[half:]
    got = np.array(ev.lower(ev.rotate_columns(m, 3))[0])
    assert np.array_equal(got[:half], np.roll(row0, 3)) and np.array_equal(got[half:], np.roll(row1, 3))
    got = np.array(ev.lower(ev.rotate_columns(m, -5))[0])
    assert np.array_equal(got[:half], np.roll(row0, -5))
    got = np.array(ev.lower(ev.rotate_rows(m))[0])
    assert np.array_equal(got, np.concatenate([row1, row0]))
    got = np.array(ev.lower(ev.rotate_bundle(m, 100))[0])
    assert np.array_equal(got[:half], np.roll(row0, 100))
    c = ev.counters()
    # popcount(3) + popcount(5) + 1 bundle; one row rotation
    assert (c["rot_cols"], c["rot_rows"]) == (5, 1)
    same = ev.rotate_columns(m, 0)  # no-op, shares the payload, counts nothing
    assert ev.counters()["rot_cols"] == 5 and ev.lower(same) == ev.lower(m)
    with pytest.raises(ValueError):
        ev.rotate_columns(m, half)


def test_rotation_direction_matches_reference_backend(dev):
    n = dev.n
    t = dev.params.t[0]
    vals = np.arange(n, dtype=np.int64) * 7 - 1000
    want = R.eval_rotate(t, n, vals, 9, rows=False, ring=True)
    ev = Evaluator(EvalContext(dev))
    got = np.array(ev.lower(ev.rotate_columns(ev.lift(vals), 9))[0])
    assert np.array_equal(got, want)


def test_mask_validates_and_counts(dev):
    ev = Evaluator(EvalContext(dev))
    m = ev.lift([4, 5, 6])
    r = ev.mask(m, [1, 0, 1])
    assert ev.lower(r)[0][:3] == [4, 0, 6]
    with pytest.raises(ValueError):
        ev.mask(m, [2])
    with pytest.raises(ValueError):
        ev.mask(m, [0, 0])
    c = ev.counters()
    assert (c["mask_mul"], c["ct_plain_mul"]) == (1, 1)


def test_fork_absorb_and_per_message_batches(dev):
    ev = Evaluator(EvalContext(dev, batch=2))
    m = ev.lift([[1, 2], [30, 40]], per_message=True)
    child = ev.fork()
    r = child.add(m, m)
    assert [row[:2] for row in ev.lower(r)] == [[2, 4], [60, 80]]
    assert ev.counters()["add"] == 0
    ev.absorb(child)
    assert ev.counters()["add"] == 1
