"""Generate the golden parity fixtures from the UNMODIFIED reference.

Run in the build container (needs /root/reference, via oracle/_ref/libbicseek_ref.so
and oracle/_ref/run_ref built by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every expected value below is computed by the reference's own code
(trend.cpp:48-72 evaluate_population / supporting_rows, datagen.cpp
gen_background / gen_scenario, evolution.cpp init_population / run).  The
fixtures are small and committed; they travel to the GPU box, where the
reference tree does not exist.
"""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))

import oracle  # noqa: E402


def _counts_and_rows(m, cols, offs, approx, neg, rows_for=None):
    mat = oracle.RefMatrix(m)
    pop = oracle.RefPopulation(cols, offs)
    counts = oracle.ref_evaluate(mat, pop, approx, neg, None)
    n = offs.size - 1
    idx = range(n) if rows_for is None else rows_for
    rows, roffs = [], [0]
    for i in idx:
        r = oracle.ref_supporting_rows(mat, cols[offs[i]:offs[i + 1]], approx, neg)
        rows.append(r)
        roffs.append(roffs[-1] + r.size)
    rows = np.concatenate(rows) if rows else np.zeros(0, np.uint32)
    return counts, np.array(list(idx), dtype=np.uint32), rows.astype(np.uint32), np.array(roffs, dtype=np.uint64)


def case(name, m, cols, offs, settings, rows_for=None):
    out = {"matrix": np.ascontiguousarray(m, dtype=np.float64), "cols": cols.astype(np.uint32),
           "offsets": offs.astype(np.uint32)}
    meta = []
    for k, (approx, neg) in enumerate(settings):
        counts, ridx, rows, roffs = _counts_and_rows(m, cols, offs, approx, neg, rows_for)
        out[f"counts_{k}"] = counts
        out[f"rows_idx_{k}"] = ridx
        out[f"rows_{k}"] = rows
        out[f"rows_offsets_{k}"] = roffs
        meta.append({"approx": approx, "negative": neg})
    out["settings"] = np.array(json.dumps(meta))
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: matrix {m.shape}, {offs.size - 1} candidates, settings {meta}")


def edge_matrix(rng):
    """Values that stress the exactness argument: ties, +-0, subnormals (f32 and
    f64), huge magnitudes, values one ulp apart, f32-exact and not."""
    f32_tiny = np.float32(1.4e-45)
    specials = np.array([
        0.0, -0.0, 1.0, -1.0, 1.0 + 2**-23, 1.0 - 2**-24, 1.0 + 2**-52, float(f32_tiny), -float(f32_tiny),
        2**-126, -2**-126, 2**-149 * 3, 3.4e38, -3.4e38, 1e-300, -1e-300, 1e300, 0.5, 0.97, 1.03,
        100.0, 97.0, 103.0, 1e-40, 7.0, 7.0, -7.0, 2.0, 2.0 * (1 - 0.03), 2.0 * (1 - 0.03) + 2**-50,
    ])
    m = rng.choice(specials, size=(64, 24))
    # rows that are exact trends / near-ties under approx in {0.03, 0.25}
    for r in range(0, 64, 4):
        base = rng.standard_normal()
        m[r, :] = base * np.cumprod(np.full(24, 1.0 - 0.03))
    return m


def main():
    if not oracle.reference_available():
        raise SystemExit("oracle/_ref/libbicseek_ref.so missing: run `make -C oracle ref` first")
    rng = np.random.default_rng(2105_01196)

    # --- test_trend.cpp:157-174: 100x20 seed 104, 50 chromosomes from Rng(12), approx 0.03
    m = oracle.ref_gen_background(100, 20, 104)
    cols, offs = oracle.ref_test_chromosomes(12, 50, 20)
    case("ref_test_pop104", m, cols, offs, [(0.03, False), (0.03, True), (0.0, False)])

    # --- test_trend.cpp:176-188: 80x16 seed 105, 37 chromosomes from Rng(13), approx 0.01 + negatives
    m = oracle.ref_gen_background(80, 16, 105)
    cols, offs = oracle.ref_test_chromosomes(13, 37, 16)
    case("ref_test_pop105", m, cols, offs, [(0.01, True), (0.01, False)])

    # --- test_trend.cpp:60-89 hand vectors (3x3 etc.) as a population over one matrix
    m = np.array([[1.0, 2.0, 3.0], [3.0, 2.0, 1.0], [2.0, 1.0, 3.0]])
    seqs = [[0, 1, 2], [2, 1, 0], [1, 2, 0], [2, 0, 1], [0, 1], [1, 0], [0, 2], [0], [0, 0, 1]]
    offs = np.cumsum([0] + [len(s) for s in seqs]).astype(np.uint32)
    cols = np.array([c for s in seqs for c in s], dtype=np.uint32)
    case("ref_hand_3x3", m, cols, offs, [(0.0, False), (0.0, True), (0.05, False), (0.5, True)])

    # --- BASELINE config 1: 500x100, 3 planted 50x8 trends, seed 1, f32-quantised; P=400 seed 42
    m = oracle.ref_gen_scenario(500, 100, 50, 8, 3, seed=1, quantize=True)
    cols, offs = oracle.ref_init_population(400, 100, seed=42)
    case("cfg1_init_pop", m, cols, offs, [(0.03, False), (0.03, True), (0.0, False), (0.2, True)],
         rows_for=list(range(0, 400, 20)))

    # --- long and short sequences, duplicates, L=1 on a quantised background (not f32: stays f64)
    m = oracle.ref_gen_background(300, 120, 7)
    seqs = [list(rng.choice(120, size=L, replace=False)) for L in (1, 2, 3, 5, 8, 17, 33, 64, 65, 100, 120)]
    seqs += [[5, 5], [3, 9, 3], [0, 1, 0, 1]]
    offs = np.cumsum([0] + [len(s) for s in seqs]).astype(np.uint32)
    cols = np.array([c for s in seqs for c in s], dtype=np.uint32)
    case("long_seqs_f64", m, cols, offs, [(0.0, False), (0.03, True), (0.5, True)])
    mq = oracle.ref_gen_background(300, 120, 7, quantize=True)
    case("long_seqs_f32", mq, cols, offs, [(0.0, True), (0.03, False), (0.9, True)])

    # --- exactness edge values
    m = edge_matrix(rng)
    seqs = [list(rng.choice(24, size=int(rng.integers(2, 9)), replace=False)) for _ in range(300)]
    offs = np.cumsum([0] + [len(s) for s in seqs]).astype(np.uint32)
    cols = np.array([c for s in seqs for c in s], dtype=np.uint32)
    case("edge_values_f64", m, cols, offs, [(0.0, True), (0.03, True), (0.25, False), (0.999, True)])
    mq = np.where(np.abs(m) < 3.4e38, m, np.sign(m) * 3.4e38).astype(np.float32).astype(np.float64)
    case("edge_values_f32", mq, cols, offs, [(0.0, True), (0.03, True), (0.25, False), (0.999, True),
                                            (2**-30, True), (0.1, True)])

    # --- fitness (trend.cpp:74-79)
    L = oracle.reference()
    fit = []
    for count in (0, 1, 5, 9, 10, 11, 100, 12345):
        for ncols in (1, 2, 3, 8, 9, 50):
            for min_rows, cap in ((10, 8), (2, 16), (2, 2)):
                fit.append((count, ncols, min_rows, cap, L.ref_fitness(count, ncols, min_rows, cap)))
    np.save(HERE / "fitness.npy", np.array(fit, dtype=np.float64))

    # --- full run() on config 1 (default: tabu stop at gen 25; forced 200 generations)
    runs = {}
    for label, extra in (("default", []), ("forced200", ["--tabu", "1000000000000"]),
                         ("neg_forced60", ["--tabu", "1000000000000", "--iters", "60", "--negative", "1"])):
        out = subprocess.run([str(REPO / "oracle" / "_ref" / "run_ref"), *extra], check=True,
                             capture_output=True, text=True).stdout
        rec = json.loads(out)
        rec.pop("wall_s")
        rec["args"] = extra
        runs[label] = rec
    (HERE / "run_cfg1.json").write_text(json.dumps(runs, indent=1, sort_keys=True) + "\n")
    print("run_cfg1.json:", {k: (v["generations"], v["termination"]) for k, v in runs.items()})


if __name__ == "__main__":
    main()
