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


def test_multi_gpu_request_fails_loudly_without_gpus():
    """--gpus N launches N ranks itself (no WORLD_SIZE): with fewer visible GPUs
    it must refuse, not time one process and report n_gpus=1."""
    import torch

    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    res = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=REPO)
    assert res.returncode == 2, (res.stdout, res.stderr)
    assert "needs 2 visible GPUs" in res.stderr
    assert not [l for l in res.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus():
    import os

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=REPO, env=env)
    assert res.returncode == 2 and "WORLD_SIZE=1 but --gpus 2" in res.stderr


@pytest.mark.gpu
def test_two_rank_rows_sharded_line():
    """The N > 1 default (row-sharded C-config, pipelined peer-memory exchange)
    run as 2 ranks sharing the box's GPU: the line reports n_gpus=2, strong
    scaling, per-rank kernel / exchange times, and the exchange-window sums
    equal the process-group all_reduce of the partial counts."""
    d = _run(["--gpus", "2", "--share-gpu", "--config", "c2", "--steps", "3", "--warmup", "3"], timeout=1200)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["shard"] == "rows"
    assert d["config"]["exchange"] == "p2p" and d["parity_device_vs_host_api"] is True
    pr = d["per_rank"]
    assert len(pr) == 2 and all(r["kernel_us"] > 0 and r["exchange_us"] >= 0 for r in pr)
    assert pr[0]["rows"] == [0, 5000] and pr[1]["rows"] == [5000, 10000]
    assert d["roofline"]["frac"] < 1.5 and d["e2e"]["value"] > 0
