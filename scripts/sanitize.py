"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family once -- upload (check + transpose), rank-plane
build, pair-trend index build + both index kernels (warp per candidate for
short vectors, CTA per candidate for long; counts and MASK), the slab kernels
(packed pairs with position-indexed counts, 32-bit plane words, + MASK), the
value kernels (f32 filter, f64, native), row scatter, single-row check; the
zero-copy host path (page-locked in/out), the marshaller and the device API.
Round 2: the lazy index (short vectors built inside the TMA kernel; long
vectors through the claim / build / count / deferred kernels, with a pool too
small for the batch), the lane-group kernel, the software-pipelined
multi-pass kernel (full and lazy), small batches read in place, and the
staged upload of a pageable matrix; the lazy index's build-first route
(claim, slab-staged build at 512 and 1024 threads, publish)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2105_01196_b200 import Evaluator, Population, TrendParams, synth  # noqa: E402
from paper_2105_01196_b200._lib import (EBIC_PATH_AUTO, EBIC_PATH_LAZY, EBIC_PATH_PLANE,  # noqa: E402
                                        EBIC_PATH_PLANE_U32, EBIC_PATH_TABLE, EBIC_PATH_VALUE)


def pinned(a):
    t = torch.empty(max(a.size, 1), dtype=torch.int32, pin_memory=True)
    v = t.numpy().view(np.uint32)[: a.size]
    v[:] = a
    return t, v


rng = np.random.default_rng(0)
ev = Evaluator(0)
ok = True
keep = []
for R, Cn in ((700, 40), (300, 700), (257, 1500), (5000, 30), (40000, 12)):
    m = rng.standard_normal((R, Cn)).astype(np.float32)
    pop = synth.random_population(200, Cn, 2, min(9, Cn), seed=1)
    paths = (EBIC_PATH_AUTO, EBIC_PATH_TABLE, EBIC_PATH_PLANE, EBIC_PATH_PLANE_U32, EBIC_PATH_VALUE)
    for path in paths if R < 40000 else (EBIC_PATH_TABLE,):
        ev.set_path(path)
        for mat in (m, m.astype(np.float64) + 1e-12):  # f32 store, then a non-f32-exact f64 store
            ev.upload(mat)
            for approx, neg in ((0.03, True), (0.0, False)):
                want = oracle.evaluate_population(mat, pop.cols, pop.offsets, approx, neg)
                got = ev.evaluate_population(pop, TrendParams(approx, neg))  # marshaller (pageable)
                ok &= np.array_equal(got, want)
                # zero-copy host path: one page-locked [offsets | cols] block, page-locked output
                tb, blk = pinned(np.concatenate([pop.offsets, pop.cols]))
                to, out = pinned(np.zeros(len(pop), np.uint32))
                keep += [tb, to]
                ppop = Population(blk[pop.offsets.size:], blk[: pop.offsets.size])
                ok &= np.array_equal(ev.evaluate_population(ppop, TrendParams(approx, neg), out=out), want)
                # device API
                d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
                d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
                d_n = torch.zeros(len(pop), dtype=torch.int32, device="cuda")
                ev.evaluate_population_device(d_c.data_ptr(), d_o.data_ptr(), len(pop), d_n.data_ptr(),
                                              TrendParams(approx, neg))
                ev.sync()
                ok &= np.array_equal(d_n.cpu().numpy().view(np.uint32), want)
                rows = ev.supporting_rows_batch(Population(pop.cols[:pop.offsets[5]], pop.offsets[:6]),
                                                TrendParams(approx, neg))
                ok &= all(np.array_equal(r, oracle.supporting_rows(mat, pop.sequence(i), approx, neg))
                          for i, r in enumerate(rows))
                ok &= ev.row_supports(3, pop.sequence(0), TrendParams(approx, neg)) == \
                    oracle.row_supports(mat, 3, pop.sequence(0), approx, neg)
ev.set_path(EBIC_PATH_AUTO)

# round 2: lazy index (short / long vectors, tiny pool), lane groups, pipelined
# multi-pass kernel (>= 32 candidates per SM), staged upload (>= 32 MB pageable)
for R, Cn, P in ((5000, 60, 300), (40000, 40, 5000)):
    m = rng.standard_normal((R, Cn)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)
    pop = synth.random_population(P, Cn, 2, 6, seed=2)
    for path, budget in ((EBIC_PATH_LAZY, 0), (EBIC_PATH_LAZY, Cn * Cn * 4 + 40 * (R // 8 + 512)), (EBIC_PATH_TABLE, 0)):
        ev.upload(m)
        ev.set_table_budget(budget)
        ev.set_path(path)
        for approx, neg in ((0.03, False), (0.03, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            for _ in range(2):  # first visit builds, the second reads the pool
                ok &= np.array_equal(ev.evaluate_population(pop, TrendParams(approx, neg)), want)
        rows = ev.supporting_rows(pop.sequence(1), TrendParams(0.03, True))
        ok &= np.array_equal(rows, oracle.supporting_rows(m, pop.sequence(1), 0.03, True))
        ev.set_table_budget(0)
        ev.set_path(EBIC_PATH_AUTO)
# the build-first route of the lazy index (claim, slab-staged build with 512
# and 1024 threads, publish) for short and long vectors, and the inline route
for R, Cn, P in ((3000, 80, 400), (40000, 40, 600), (2000, 1800, 400)):
    m = rng.standard_normal((R, Cn)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)
    m[rng.random(m.shape) < 0.05] = 0.0
    pop = synth.random_population(P, Cn, 2, 6, seed=5)
    for build in (2, 1):
        ev.upload(m)
        ev.set_path(EBIC_PATH_LAZY)
        ev.set_lazy_build(build)
        for neg in (False, True):
            ok &= np.array_equal(ev.evaluate_population(pop, TrendParams(0.03, neg)),
                                 oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, neg))
        ev.set_lazy_build(0)
        ev.set_path(EBIC_PATH_AUTO)
# small page-locked batch read in place; the lane-group kernel (R <= 4096)
m = rng.standard_normal((3000, 200)).astype(np.float32)
ev.upload(m)
pop = synth.random_population(392, 200, 2, 6, seed=3)
tb, blk = pinned(np.concatenate([pop.offsets, pop.cols]))
to, out = pinned(np.zeros(len(pop), np.uint32))
keep += [tb, to]
ppop = Population(blk[pop.offsets.size:], blk[: pop.offsets.size])
ok &= np.array_equal(ev.evaluate_population(ppop, TrendParams(0.03, False), out=out),
                     oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False))
# staged upload of a pageable f64 matrix (>= 32 MB)
big = rng.standard_normal((2100, 2000))
ev.upload(big)
pop = synth.random_population(64, 2000, 2, 5, seed=4)
ok &= np.array_equal(ev.evaluate_population(pop, TrendParams(0.03, False)),
                     oracle.evaluate_population(big, pop.cols, pop.offsets, 0.03, False))
print("sanitize workload parity:", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
