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
    # same workload description as our arm (the driver compares like with like)
    c = d["config"]
    assert c["workload"].startswith("lola-mnist") and c["images_per_gpu_per_step"] == 64 and c["n"] == 16384


def test_reference_arm_never_loads_the_device_library():
    """The reference arm's workers get parameters from params.py (pure
    Python) and run only oracle/_ref/libpackref.so."""
    code = ("import sys; sys.argv=['bench.py']; sys.path.insert(0, %r); import bench; "
            "bench._ref_init('lola-mnist', 32); bench._ref_image(0); "
            "maps = open('/proc/self/maps').read(); "
            "assert 'liblola_b200' not in maps, 'device library mapped'; assert 'libpackref' in maps; print('ok')"
            % str(ROOT))
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "ok" in p.stdout, p.stderr[-2000:]


def test_multi_gpu_request_never_measures_one_gpu():
    """--gpus N without torchrun relaunches N ranks, or fails loudly when the
    box has fewer devices (here: none); it never prints an n_gpus=1 line."""
    env = dict(os.environ, PYTHONPATH=str(ROOT), CUDA_VISIBLE_DEVICES="")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0
    assert "--gpus 2 requested" in (p.stderr + p.stdout)
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")]
    env["WORLD_SIZE"] = "3"
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=3" in p.stderr


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
    assert d["parity"]["images"] == 2 and d["parity"]["mismatches"] == 0


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
    assert d["cpu_baseline_bfv"]["value"] > 0 and d["cpu_baseline_bfv"]["seconds_per_key_switch"] > 0
    assert d["latency_ms"]["he_steps"] > 0
    w = d["value_w64"]
    assert w["value"] > 0 and w["parity"]["mismatches"] == 0 and w["dtype"] == "u64"
    assert len(d["primitives"]) == 5 and all(p["rotations_per_s"] > 0 for p in d["primitives"])
