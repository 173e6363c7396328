"""The reference's own hot-path test suite and its end-to-end run(), relinked
against the device drop-in TU (csrc/bicseek_trend_device.cpp in place of
proj/src/trend.cpp) -- the strongest drop-in evidence: UNCHANGED reference
tests and UNCHANGED evolution.cpp, running on the B200 evaluator.

The binaries are built in the build container by oracle/Makefile (`device`)
from the reference sources and travel to the GPU box prebuilt.
"""
import json
import os
import subprocess

import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu

REF = REPO / "oracle" / "_ref"


def _need(name):
    exe = REF / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (reference tree absent at build time)")
    return exe


def test_reference_test_trend_passes_on_device():
    exe = _need("test_trend_device")
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "| 0 failed" in res.stdout, res.stdout


@pytest.mark.parametrize("label", ["default", "forced200", "neg_forced60"])
def test_run_config1_byte_identical_to_reference(label):
    """BASELINE config 1: full run() (tournament, mutation/crossover, tabu list,
    top-rank archive) with device evaluation == the reference CPU run."""
    exe = _need("run_device")
    golden = json.loads((GOLDEN / "run_cfg1.json").read_text())[label]
    out = subprocess.run([str(exe), *golden["args"]], check=True, capture_output=True, text=True,
                         timeout=600).stdout
    got = json.loads(out)
    assert json.dumps(got["result"], sort_keys=True) == json.dumps(golden["result"], sort_keys=True)
    assert got["generations"] == golden["generations"]
    assert got["termination"] == golden["termination"]


def _archive_env(mode):
    env = dict(os.environ)
    env["EBIC_ARCHIVE_ROWS"] = "1" if mode == "lists" else "0"
    return env


@pytest.mark.parametrize("archive", ["overlaps", "lists"])
@pytest.mark.parametrize("label", ["default", "forced200", "neg_forced60"])
def test_device_aware_driver_byte_identical_to_reference(label, archive):
    """The device-aware evolution driver (csrc/bicseek_run_device.cpp: one upload
    per run, evaluation overlapped with breeding, batched archive row data --
    device-side overlap counts by default, host row lists with
    EBIC_ARCHIVE_ROWS=1) returns exactly the reference run()'s result on
    BASELINE config 1."""
    exe = _need("run_device_overlap")
    golden = json.loads((GOLDEN / "run_cfg1.json").read_text())[label]
    out = subprocess.run([str(exe), "--engine", "device", *golden["args"]], check=True, capture_output=True,
                         text=True, timeout=600, env=_archive_env(archive)).stdout
    got = json.loads(out)
    assert json.dumps(got["result"], sort_keys=True) == json.dumps(golden["result"], sort_keys=True)
    assert got["generations"] == golden["generations"]
    assert got["termination"] == golden["termination"]


@pytest.mark.parametrize("archive", ["overlaps", "lists"])
def test_device_aware_driver_matches_reference_at_scale(archive):
    """A larger run (10k x 500, P=1024, 15 generations, negatives on): the
    driver's output equals the unchanged reference GA on the device TU."""
    exe_a, exe_b = _need("run_device"), _need("run_device_overlap")
    args = ["--rows", "10000", "--cols", "500", "--bic-rows", "500", "--bic-cols", "20", "--pop", "1024",
            "--iters", "15", "--tabu", "1000000000000", "--negative", "1"]
    a = json.loads(subprocess.run([str(exe_a), *args], check=True, capture_output=True, text=True,
                                  timeout=600).stdout)
    b = json.loads(subprocess.run([str(exe_b), "--engine", "device", *args], check=True, capture_output=True,
                                  text=True, timeout=600, env=_archive_env(archive)).stdout)
    assert a["result"] == b["result"] and a["generations"] == b["generations"]


def test_concurrent_runs_one_context_per_thread():
    """bench --jobs style: four independent datasets, one unchanged run() per
    thread; every thread's drop-in TU gets its own device context (spread
    round-robin over the visible GPUs -- dataset-level multi-GPU).  Each job's
    result equals the reference CPU build's."""
    exe_ref, exe_dev = _need("run_ref"), _need("run_device")
    args = ["--jobs", "4", "--rows", "2000", "--cols", "200", "--bic-rows", "200", "--bic-cols", "10",
            "--pop", "512", "--iters", "30", "--tabu", "1000000000000"]
    want = subprocess.run([str(exe_ref), *args], check=True, capture_output=True, text=True, timeout=600).stdout
    got = subprocess.run([str(exe_dev), *args], check=True, capture_output=True, text=True, timeout=600).stdout
    want_l, got_l = want.strip().splitlines(), got.strip().splitlines()
    assert len(got_l) == len(want_l) == 4
    for a, b in zip(want_l, got_l):
        assert json.loads(a) == json.loads(b)


NONDEFAULT = {
    "overlap_0.3": ["--overlap", "0.3"],
    "tournament9_crossover_heavy": ["--tournament", "9", "--weights", "0.05,0.05,0.1,0.1,0.7"],
    "six_biclusters_two_elites": ["--biclusters", "6", "--elite", "2"],
    "penalty2_approx0.1_neg": ["--penalty", "2.0", "--approx", "0.1", "--negative", "1"],
}


@pytest.mark.parametrize("label", sorted(NONDEFAULT))
def test_run_nondefault_params_byte_identical(label):
    """run() with non-default GA parameters (evolution.hpp:20-39: overlap
    threshold, tournament size, crossover-heavy operator weights, bicluster
    count, elites, crowding penalty, approx/negatives): the unchanged reference
    GA on the drop-in TU (default environment: the cached matrix verified on
    every call) and the device-aware driver (bicseek_run_device.cpp, its own
    restatement of the archive and breeding loop) both equal the reference CPU
    build, result, generations and termination."""
    exe_ref, exe_dev, exe_drv = _need("run_ref"), _need("run_device"), _need("run_device_overlap")
    args = ["--rows", "2000", "--cols", "150", "--bic-rows", "120", "--bic-cols", "10", "--num-bics", "3",
            "--pop", "600", "--iters", "40", "--tabu", "1000000000000", *NONDEFAULT[label]]
    env = dict(os.environ)
    env.pop("EBIC_SHIM_TRUST_POINTER", None)
    want = json.loads(subprocess.run([str(exe_ref), *args], check=True, capture_output=True, text=True,
                                     timeout=600).stdout)
    for exe, extra in ((exe_dev, []), (exe_drv, ["--engine", "device"])):
        got = json.loads(subprocess.run([str(exe), *extra, *args], check=True, capture_output=True, text=True,
                                        timeout=600, env=env).stdout)
        assert got["result"] == want["result"], (exe.name, label)
        assert got["generations"] == want["generations"] and got["termination"] == want["termination"]
