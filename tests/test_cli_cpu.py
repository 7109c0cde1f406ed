"""The reference CLI builds here (CLI11 stand-in) and runs on the manifest
and IDX files the tests write: `packnn infer --backend ring` gives the
reference integer oracle's class and scores; the B200 CLI refuses the
reference's CPU backends with the CLI's usage exit code."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from oracle import refbind as R
from paper_1812_10659_b200 import nets
from cli_files import write_idx, write_model

ROOT = Path(__file__).resolve().parents[1]
REF_CLI = ROOT / "oracle" / "_ref" / "packnn"
B200_CLI = ROOT / "oracle" / "_ref" / "packnn_b200"


@pytest.fixture
def files(tmp_path):
    if not REF_CLI.exists():
        pytest.skip("oracle/_ref/packnn not built")
    net = nets.toy_net()
    model = write_model(net, tmp_path / "toy.json")
    imgs = nets.images(9, net, 3)
    idx = write_idx(imgs, net.input_shape[1:], tmp_path / "toy.idx")
    return net, imgs, model, idx


def test_reference_cli_ring_backend_on_written_files(files):
    net, imgs, model, idx = files
    for i in range(3):
        p = subprocess.run([str(REF_CLI), "infer", "--model", str(model), "--input", str(idx), "--plan", "lola-mnist",
                            "--backend", "ring", "--n", "4096", "--index", str(i)], capture_output=True, text=True,
                           timeout=300)
        assert p.returncode == 0, p.stderr
        scores = [int(v) for v in p.stdout.split("scores")[1].split()]
        assert scores == R.forward_integer(net, imgs[i])
        assert p.stdout.startswith(f"class {max(range(len(scores)), key=lambda k: (scores[k], -k))}")


def test_b200_cli_usage_errors(files):
    _, _, model, idx = files
    p = subprocess.run([str(B200_CLI), "infer", "--model", str(model), "--input", str(idx), "--backend", "cpu"],
                       capture_output=True, text=True, timeout=60)
    assert p.returncode == 2 and "not in" in p.stderr
    p = subprocess.run([str(B200_CLI), "infer", "--input", str(idx)], capture_output=True, text=True, timeout=60)
    assert p.returncode == 2 and "--model is required" in p.stderr
