"""`packnn infer --backend gpu`: the reference's own CLI
(proj/src/cli.cpp, tools/main.cpp, model_io.cpp) built with the two-line
backend change and linked with the B200 evaluator (oracle/_ref/packnn_b200),
on a model manifest + IDX input written in the reference's formats. Its
output (predicted class and every score) equals the unmodified reference CLI
(oracle/_ref/packnn) with `--backend ring` on the same files."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from paper_1812_10659_b200 import nets
from cli_files import write_idx, write_model

ROOT = Path(__file__).resolve().parents[1]
REF_CLI = ROOT / "oracle" / "_ref" / "packnn"
B200_CLI = ROOT / "oracle" / "_ref" / "packnn_b200"


def _infer(cli, model, idx, backend, extra, index=0):
    p = subprocess.run([str(cli), "infer", "--model", str(model), "--input", str(idx), "--plan", "lola-mnist",
                        "--backend", backend, "--index", str(index), *extra], capture_output=True, text=True,
                       timeout=600)
    return p.returncode, p.stdout, p.stderr


def _files(tmp_path, net, cfg, count):
    model = write_model(net, tmp_path / "model.json")
    idx = write_idx(nets.images(cfg, net, count), net.input_shape[1:] if net.input_shape[0] == 1 else net.input_shape,
                    tmp_path / "inputs.idx")
    return model, idx


@pytest.mark.parametrize("which", ["toy", "lola-mnist-cfg0"])
@pytest.mark.gpu
def test_backend_gpu_matches_reference_cli(tmp_path, which):
    if which == "toy":
        net, cfg, extra = nets.toy_net(), 9, ["--n", "4096"]
    else:
        from paper_1812_10659_b200.params import SUGGESTED_PLAIN_PRIMES

        net, cfg = nets.lola_mnist_net(config=0), 0
        extra = ["--n", "16384", "--primes", ",".join(str(p) for p in SUGGESTED_PLAIN_PRIMES[:5])]
    model, idx = _files(tmp_path, net, cfg, 2)
    for i in range(2):
        rc_r, out_r, err_r = _infer(REF_CLI, model, idx, "ring", extra, i)
        assert rc_r == 0, err_r
        rc_g, out_g, err_g = _infer(B200_CLI, model, idx, "gpu", extra, i)
        assert rc_g == 0, err_g
        assert out_g == out_r and out_g.startswith("class ")
        assert "backend gpu" in err_g
