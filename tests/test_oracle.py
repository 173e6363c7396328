"""The oracle is pinned before it is trusted (CPU only).

* the C restatement (oracle/liboracle.so) vs the golden fixtures produced by the
  unmodified reference (tests/golden/make_golden.py);
* vs the hand vectors of proj/tests/test_trend.cpp:60-89;
* vs the live reference library on random inputs (when oracle/_ref is built);
* the reference's own doctest suites, compiled unchanged against the shim.
"""
import subprocess

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, REPO, golden_cases, load_golden


@pytest.mark.parametrize("name", golden_cases())
def test_port_matches_reference_golden(name):
    z, settings = load_golden(name)
    m, cols, offs = z["matrix"], z["cols"], z["offsets"]
    for k, s in enumerate(settings):
        got = oracle.evaluate_population(m, cols, offs, s["approx"], s["negative"], threads=2)
        np.testing.assert_array_equal(got, z[f"counts_{k}"], err_msg=f"{name} setting {s}")
        ro = z[f"rows_offsets_{k}"]
        for j, i in enumerate(z[f"rows_idx_{k}"]):
            rows = oracle.supporting_rows(m, cols[offs[i]:offs[i + 1]], s["approx"], s["negative"])
            np.testing.assert_array_equal(rows, z[f"rows_{k}"][ro[j]:ro[j + 1]])


def test_port_f32_path_matches_f64_path_on_quantised_matrix():
    z, settings = load_golden("cfg1_init_pop")
    m32 = z["matrix"].astype(np.float32)
    assert np.array_equal(m32.astype(np.float64), z["matrix"])
    for k, s in enumerate(settings):
        got = oracle.evaluate_population(m32, z["cols"], z["offsets"], s["approx"], s["negative"])
        np.testing.assert_array_equal(got, z[f"counts_{k}"])


def test_port_hand_vectors():
    # test_trend.cpp:60-89
    rs = oracle.row_supports
    assert rs(np.array([[1.0, 2.0, 3.0]]), 0, [0, 1, 2], 0.0, False)
    assert not rs(np.array([[1.0, 2.0, 3.0]]), 0, [2, 1, 0], 0.0, False)
    assert rs(np.array([[3.0, 1.0, 2.0]]), 0, [1, 2, 0], 0.0, False)
    assert not rs(np.array([[1.0, 1.0]]), 0, [0, 1], 0.0, False)
    assert rs(np.array([[1.0, 1.0]]), 0, [0, 1], 0.05, False)
    assert not rs(np.array([[2.0, 2.0, 2.0]]), 0, [0, 1, 2], 0.0, True)
    m = np.array([[1.0, 2.0, 3.0], [3.0, 2.0, 1.0], [2.0, 1.0, 3.0]])
    assert list(oracle.supporting_rows(m, [0, 1, 2], 0.0, False)) == [0]
    assert list(oracle.supporting_rows(m, [0, 1, 2], 0.0, True)) == [0, 1]
    assert list(oracle.supporting_rows(m, [2, 0, 1], 0.0, False)) == []


def test_port_fitness_golden():
    fit = np.load(GOLDEN / "fitness.npy")
    for count, ncols, min_rows, cap, expect in fit:
        assert oracle.fitness(int(count), int(ncols), int(min_rows), int(cap)) == expect


def test_port_thread_count_invariance():
    # test_trend.cpp:176-188 (worker-count invariance)
    z, _ = load_golden("ref_test_pop105")
    seq = oracle.evaluate_population(z["matrix"], z["cols"], z["offsets"], 0.01, True, threads=1)
    for t in (2, 3, 8):
        np.testing.assert_array_equal(
            oracle.evaluate_population(z["matrix"], z["cols"], z["offsets"], 0.01, True, threads=t), seq)


needs_ref = pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_vs_live_reference_random(seed):
    rng = np.random.default_rng(seed)
    R, Cn = int(rng.integers(1, 400)), int(rng.integers(2, 60))
    m = oracle.ref_gen_background(R, Cn, seed, quantize=bool(seed % 2))
    m[rng.random(m.shape) < 0.05] = 0.0  # ties
    seqs = [rng.choice(Cn, size=int(rng.integers(1, min(Cn, 12) + 1)), replace=False) for _ in range(200)]
    offs = np.cumsum([0] + [len(s) for s in seqs]).astype(np.uint32)
    cols = np.concatenate(seqs).astype(np.uint32)
    mat, pop = oracle.RefMatrix(m), oracle.RefPopulation(cols, offs)
    for approx in (0.0, float(rng.uniform(0, 0.3)), 0.999):
        for neg in (False, True):
            ref = oracle.ref_evaluate(mat, pop, approx, neg, oracle.RefPool(4))
            np.testing.assert_array_equal(oracle.evaluate_population(m, cols, offs, approx, neg), ref)
            i = int(rng.integers(len(seqs)))
            np.testing.assert_array_equal(oracle.supporting_rows(m, seqs[i], approx, neg),
                                          oracle.ref_supporting_rows(mat, seqs[i], approx, neg))


@needs_ref
@pytest.mark.parametrize("suite", ["core", "trend", "metrics"])
def test_reference_doctest_suites_pass_with_shim(suite):
    exe = REPO / "oracle" / "_ref" / f"test_{suite}_ref"
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failed" in res.stdout


@needs_ref
def test_reference_run_matches_golden():
    import json

    golden = json.loads((GOLDEN / "run_cfg1.json").read_text())
    for label, rec in golden.items():
        out = subprocess.run([str(REPO / "oracle" / "_ref" / "run_ref"), *rec["args"]], check=True,
                             capture_output=True, text=True, timeout=300).stdout
        got = json.loads(out)
        got.pop("wall_s")
        assert got["result"] == rec["result"] and got["generations"] == rec["generations"]
        assert got["termination"] == rec["termination"]
