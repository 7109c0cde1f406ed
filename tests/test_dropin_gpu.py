"""The drop-in proof: the reference's OWN plan builders,
LoLa kernels, representations and execute() — proj/src/plan.cpp,
kernels.cpp, representation.cpp compiled unmodified — running on this
repo's B200 evaluator through the C-ABI (oracle/b200_dropin/evaluator_b200.cpp
implements the unmodified proj/include/packnn/evaluator.hpp over lb_eval_*,
as a third BackendKind). Decrypted logits == forward_integer
(proj/src/layers.cpp:560-594); per-step counters == the reference's Ring
backend run; execute()'s own per-step counter check (plan.cpp:617-621)
passes on real ciphertexts."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import refbind as R
from paper_1812_10659_b200 import nets
from paper_1812_10659_b200.params import lola_small_params_w32, make_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["toy-lola-mnist", "toy-lola-dense-mnist", "lola-small"])
def test_reference_execute_on_b200_backend(which):
    import torch

    torch.cuda.init()
    if which == "lola-small":
        net, strategy, prm, cfg = nets.lola_small_net(), "lola-small", lola_small_params_w32(seed=3), 3
    else:
        net, strategy, cfg = nets.toy_net(), which[4:], 9
        prm = make_params(4096, L=7, T=3, K=1, seed=5)
    for i in range(2):
        x = nets.images(cfg, net, 1, start=i)[0]
        scores, counters = R.run_plan_b200(net, strategy, prm, x)
        assert scores == R.forward_integer(net, x), f"image {i}"
        _, ref_counters, _ = R.run_plan(net, strategy, prm.n, prm.t, x, ring=True)
        assert np.array_equal(counters, ref_counters)
