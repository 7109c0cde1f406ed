"""Shared fixtures. GPU tests are marked `gpu`; everything else runs on CPU."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a library)")


def _ensure_oracles() -> None:
    """Build the CPU oracles if missing (dev container only: the GPU box gets
    the prebuilt oracle/_ref/*.so with the repo snapshot)."""
    ref = ROOT / "oracle" / "_ref"
    need = [ref / "libbfvoracle.so"]
    if Path("/root/reference/proj/src").exists():
        need += [ref / "libpackref.so", ref / "libpackb200.so"]
    if all(p.exists() for p in need):
        return
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "-j8"], check=True)


@pytest.fixture(scope="session", autouse=True)
def oracles_built():
    _ensure_oracles()
