"""bench.py keeps the driver's JSON contract: the reference arm on CPU (it runs
the reference's own evaluate_population on the host) and, on a GPU, our arm
with the roofline / cpu_baseline / e2e / clocks objects."""
import json
import subprocess
import sys

import pytest

from conftest import REPO

import oracle

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout=900):
    res = subprocess.run([sys.executable, str(REPO / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=REPO)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c2", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "evals/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"] and "model" not in d["config"]


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "c2", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys() and r["unit"] == "GB/s"
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 * max(1.0, r["frac"])
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= cb.keys() and cb["parity_with_gpu"] is True
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()
    assert d["gpu_launches"] >= d["steps"] and d["parity_device_vs_host_api"] is True
    assert "l2" in d["config"]
