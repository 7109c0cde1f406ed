"""bench.py's JSON-line contract, for both arms.

The reference arm (`--impl reference`) runs the compiled reference
(`oracle/_ref/libpackref.so`) on host cores, so it is checked here on CPU; our
arm needs the B200 and is checked under the gpu marker with a tiny batch."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    if not (ROOT / "oracle" / "_ref" / "libpackref.so").exists():
        pytest.skip("oracle/_ref not built (run __graft_entry__.build())")
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], timeout=600)
    assert d["impl"] == "reference"
    assert BASE_KEYS <= d.keys()
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "inferences/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--no-extras", "--steps", "1", "--warmup", "3", "--batch", "2"], timeout=900)
    assert "impl" not in d or d["impl"] == "ours"
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["dtype"] in ("u32", "u64")
    assert d["config"]["workload"].startswith("lola-mnist")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != d["value"]
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


@pytest.mark.gpu
def test_our_arm_roofline_and_cpu_baseline():
    d = _run(["--steps", "1", "--warmup", "3", "--batch", "2", "--cpu-sample", "1"], timeout=900)
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    hv = r["hbm_view"]
    assert 0 < hv["frac"] < 1 and hv["algorithmic_bytes_per_launch"] > 0
    assert 0 < d["roofline_ntt"]["frac"] < 1
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] == 1 and cb["kind"] in ("reference", "port") and cb["sample"]
    assert d["latency_ms"]["he_steps"] > 0
