"""The paired kernels (two same-prime transforms per cluster: forward NTT,
ModDown, key inner product) only run on launches of LB_PAIR_MIN (32 polys) /
LB_KS_PAIR_MIN / LB_MD_PAIR_MIN (8 / 32 ciphertexts) or more. This re-runs the coefficient-exact ciphertext tests with
the threshold at 2, so every ring size, prime set and odd count goes through
them too (the oracle comparisons inside those tests are the check)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_ciphertext_tests_through_paired_kernels():
    env = dict(os.environ, LB_PAIR_MIN="2", LB_KS_PAIR_MIN="2", LB_MD_PAIR_MIN="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_bfv_gpu.py", "tests/test_sweep_batch_gpu.py",
                        "tests/test_sweep_gpu.py", "-m", "gpu", "-x", "-q"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_unpaired_inverse_transforms():
    """The single-transform inverse NTT (LB_NTT_PAIR=1: forward pairs only) is
    the fallback for small batches; this runs it on every batch size."""
    env = dict(os.environ, LB_PAIR_MIN="2", LB_KS_PAIR_MIN="2", LB_MD_PAIR_MIN="2", LB_NTT_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_bfv_gpu.py", "tests/test_sweep_gpu.py", "-m", "gpu",
                        "-x", "-q"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
