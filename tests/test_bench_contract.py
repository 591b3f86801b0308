"""bench.py keeps the driver's JSON-line contract.

CPU: the reference arm (`--impl reference`: the reference package from
baseline/_ref on the host cores, on a sample of the same workload), the
config object shared by both arms, --gpus N failing loudly without N GPUs.
GPU: the native arm on the C4 workload, short run."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(1, "weak")   # the native arm's config
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "MCUPS"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_config_shared_and_sized():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.workload_config(1, "weak")["cells"] == 256 ** 3
    assert bench.workload_config(8, "weak")["cells"] == 8 * 256 ** 3     # C5: L18
    assert bench.workload_config(8, "strong")["cells"] == 256 ** 3       # C4 over 8
    assert bench.workload_level(4, "weak") == 17 and bench.sample_np(17) == 256


def test_multi_gpu_request_fails_loudly_without_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("two GPUs visible: the spawn path would run")
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "1"], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode != 0 and "only" in out.stderr and "visible" in out.stderr


@pytest.mark.gpu
def test_native_arm_line():
    d = _run(["--steps", "3", "--warmup", "3", "--skip-cpu", "--repeats", "3"], 900)
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["higher_is_better"] is True and d["dtype"] == "f64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # a repeated call (recycled arenas) and the cold first call beside it
    assert e["cold"]["value"] > 0 and "arenas" in e and "arenas" in e["cold"]
    assert set(e["phases_s"]) >= {"blocks", "finalize", "upload", "steps", "download"}
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert "workload" in d["config"]
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.workload_config(1, "weak")
    rep = d["repeats"]
    assert rep["n"] >= 3 and len(rep["ms"]) == rep["n"] and rep["median_ms"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_native_arm_two_gpus(scaling):
    """--gpus 2 spawns two NCCL ranks itself (needs two visible GPUs)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    d = _run(["--gpus", "2", "--steps", "3", "--warmup", "3", "--skip-cpu", "--skip-e2e",
              "--scaling", scaling, "--repeats", "1"], 1200)
    sys.path.insert(0, ROOT)
    import bench
    assert d["n_gpus"] == 2 and d["config"] == bench.workload_config(2, scaling)
    assert d["scaling"] == scaling and d["comm"]["nranks"] == 2
    assert all(r["messages_per_stage"] > 0 for r in d["comm"]["per_rank"])
