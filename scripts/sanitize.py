"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once -- upload (check + transpose), rank-plane build, both
packed-pair and 32-bit slab kernels (+ MASK), value kernels (f32 filter, f64,
native), row scatter, single-row check."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2105_01196_b200 import Evaluator, Population, TrendParams, synth  # noqa: E402
from paper_2105_01196_b200._lib import EBIC_PATH_AUTO, EBIC_PATH_PLANE_U32, EBIC_PATH_VALUE  # noqa: E402

rng = np.random.default_rng(0)
ev = Evaluator(0)
ok = True
for R, Cn in ((700, 40), (300, 700), (257, 1500)):
    m = rng.standard_normal((R, Cn)).astype(np.float32)
    pop = synth.random_population(200, Cn, 2, 9, seed=1)
    for path in (EBIC_PATH_AUTO, EBIC_PATH_PLANE_U32, EBIC_PATH_VALUE):
        ev.set_path(path)
        for mat in (m, m.astype(np.float64) + 1e-12):  # f32 store, then a non-f32-exact f64 store
            ev.upload(mat)
            for approx, neg in ((0.03, True), (0.0, False)):
                got = ev.evaluate_population(pop, TrendParams(approx, neg))
                ok &= np.array_equal(got, oracle.evaluate_population(mat, pop.cols, pop.offsets, approx, neg))
                rows = ev.supporting_rows_batch(Population(pop.cols[:pop.offsets[5]], pop.offsets[:6]),
                                                TrendParams(approx, neg))
                ok &= all(np.array_equal(r, oracle.supporting_rows(mat, pop.sequence(i), approx, neg))
                          for i, r in enumerate(rows))
                ok &= ev.row_supports(3, pop.sequence(0), TrendParams(approx, neg)) == \
                    oracle.row_supports(mat, 3, pop.sequence(0), approx, neg)
ev.set_path(EBIC_PATH_AUTO)
print("sanitize workload parity:", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
