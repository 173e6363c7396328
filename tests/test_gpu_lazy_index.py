"""The lazy pair-trend index (ebic_lazy.cuh): pair vectors built by the count
kernel the first time a candidate needs them and kept in a pool.  Every count
and row list must equal the C oracle whatever the cache holds -- first use,
reuse across batches, warps racing for the same new pair, a pool too small for
the batch (private builds), pool growth and resets, approx changes, f32 and
f64 stores -- and AUTO must move to the full index once half the pairs were
built (ski rental) or when asked (ebic_matrix_prepare)."""
import numpy as np
import pytest

import oracle
from paper_2105_01196_b200 import EBIC_STORE_F64, Population, TrendParams, synth
from paper_2105_01196_b200._lib import EBIC_PATH_AUTO, EBIC_PATH_LAZY

pytestmark = pytest.mark.gpu

SETTINGS = ((0.03, False), (0.0, True), (0.25, True), (0.03, True))


def _matrix(R, C, seed, f64=False):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((R, C)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)
    m[rng.random(m.shape) < 0.03] = 0.0
    if f64:
        m = m.astype(np.float64)
        m[::7, ::3] += 1e-9  # not float32-representable: a float64 store
    return m


def _pop(C, n, seed, dup_pairs=False):
    rng = np.random.default_rng(seed)
    seqs = [rng.choice(C, size=int(rng.integers(1, min(C, 9) + 1)), replace=False) for _ in range(n)]
    seqs += [rng.integers(0, C, size=int(rng.integers(2, 6))) for _ in range(n // 10)]  # duplicate columns
    seqs += [rng.choice(C, size=min(C, 40), replace=False)]  # > 32 pairs: lookups past the lanes
    if dup_pairs:  # many candidates sharing the same few pairs: warps race to build them
        seqs += [[3, 5, 7, 3 + (k % 2)] for k in range(400)]
    return Population.from_sequences(seqs)


# R > 32768: long vectors (> 256 slices) -- claim / build kernels ahead of the
# multi-pass count kernel instead of builds inside the TMA kernel
@pytest.mark.parametrize("R", [1, 33, 1000, 4099, 20000, 32768, 32769, 70001])
@pytest.mark.parametrize("f64", [False, True])
@pytest.mark.parametrize("build", [0, 1, 2], ids=["auto", "inline", "first"])
def test_lazy_index_vs_oracle(evaluator, R, f64, build):
    """Every build route of the lazy index (auto; inside the count kernel;
    the slab build pass ahead of it) against the oracle."""
    C = 150
    m = _matrix(R, C, R + 7 * f64, f64)
    store = evaluator.upload(m)
    assert (store == EBIC_STORE_F64) == f64
    evaluator.set_path(EBIC_PATH_LAZY)
    evaluator.set_lazy_build(build)
    try:
        for batch in range(3):  # first use, then reuse (and new pairs) across batches
            pop = _pop(C, 700, seed=batch, dup_pairs=batch == 1)
            for approx, neg in SETTINGS:
                want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
                got = evaluator.evaluate_population(pop, TrendParams(approx, neg))
                np.testing.assert_array_equal(got, want, err_msg=f"R={R} batch={batch} approx={approx} neg={neg}")
            assert evaluator.index_stats()["mode"] == "lazy"
        for j in (0, 5, len(pop) - 1):
            for approx, neg in ((0.03, False), (0.1, True)):
                rows = evaluator.supporting_rows(pop.sequence(j), TrendParams(approx, neg))
                np.testing.assert_array_equal(rows, oracle.supporting_rows(m, pop.sequence(j), approx, neg))
        st = evaluator.index_stats()
        assert st["lazy_slots_cap"] > 0 and st["lazy_bytes"] > 0
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)
        evaluator.set_lazy_build(0)


@pytest.mark.parametrize("R", [9000, 40000])
@pytest.mark.parametrize("build", [0, 2], ids=["auto", "first"])
def test_lazy_pool_too_small_resets_and_private_builds(evaluator, R, build):
    """A budget that holds only a few dozen pair vectors: most new pairs find
    no slot (private builds; for long vectors, slices computed by the count
    kernel), the pool starts over; counts stay exact."""
    C = 200
    m = _matrix(R, C, 3)
    evaluator.upload(m)
    wp = ((R + 31) // 32 + 127) // 128 * 128 if (R + 31) // 32 > 128 else ((R + 31) // 32 + 3) // 4 * 4
    evaluator.set_table_budget(C * C * 4 + 40 * wp * 4)
    evaluator.set_path(EBIC_PATH_LAZY)
    evaluator.set_lazy_build(build)
    try:
        for batch in range(6):
            pop = _pop(C, 500, seed=100 + batch, dup_pairs=True)
            for approx, neg in ((0.03, False), (0.03, True)):
                want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
                got = evaluator.evaluate_population(pop, TrendParams(approx, neg))
                np.testing.assert_array_equal(got, want, err_msg=f"batch {batch} neg {neg}")
        st = evaluator.index_stats()
        assert st["lazy_slots_cap"] <= 40 and st["lazy_resets"] >= 1
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)
        evaluator.set_table_budget(0)
        evaluator.set_lazy_build(0)


@pytest.mark.parametrize("R,n_streams,build", [(12000, 1, 0), (40000, 1, 0), (40000, 2, 0), (12000, 2, 0),
                                                (12000, 2, 1), (12000, 2, 2), (12000, 1, 2)])
def test_lazy_device_api_back_to_back(evaluator, R, n_streams, build):
    """Device-pointer batches issued back to back (no host sync, programmatic
    dependent launch, the host's view of the pool lagging): exact.  With two
    streams, batches claim and build concurrently (the batch tags keep each
    build kernel to its own slots; a pair another stream is building is built
    privately by the count kernel)."""
    torch = pytest.importorskip("torch")
    C = 400
    m = _matrix(R, C, 11)
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_LAZY)
    evaluator.set_lazy_build(build)
    try:
        pops = [synth.random_population(5000, C, 2, 8, seed=300 + k) for k in range(6)]
        want = [oracle.evaluate_population(m, p.cols, p.offsets, 0.03, True) for p in pops]
        dev = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda())
               for p in pops]
        outs = [torch.full((5000,), -1, dtype=torch.int32, device="cuda") for _ in range(18)]
        streams = [torch.cuda.Stream() for _ in range(n_streams)]
        torch.cuda.synchronize()
        for i in range(18):
            dc, do = dev[i % 6]
            evaluator.evaluate_population_device(dc.data_ptr(), do.data_ptr(), 5000, outs[i].data_ptr(),
                                                 TrendParams(0.03, True), stream=streams[i % n_streams].cuda_stream)
        for s in streams:
            s.synchronize()
        evaluator.sync()
        for i in range(18):
            np.testing.assert_array_equal(outs[i].cpu().numpy().view(np.uint32), want[i % 6], err_msg=f"launch {i}")
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)
        evaluator.set_lazy_build(0)


def test_auto_policy_lazy_then_full(evaluator):
    """AUTO on a matrix whose full index is large (> 1 GiB): the first batches
    run on the lazy index (no full build on the first call); once half of the
    C^2 pairs were built lazily the full index is bought (ski rental); an
    explicit prepare() builds the full index at once."""
    R, C = 20000, 1000  # full index 2.56 GB
    m = _matrix(R, C, 17)
    evaluator.upload(m)
    pop0 = synth.random_population(16384, C, 3, 5, seed=1)
    want0 = oracle.evaluate_population(m, pop0.cols, pop0.offsets, 0.03, False)
    np.testing.assert_array_equal(evaluator.evaluate_population(pop0, TrendParams()), want0)
    st = evaluator.index_stats()
    assert st["mode"] == "lazy" and st["full_bytes"] == 0
    mode = "lazy"
    for k in range(40):
        pop = synth.random_population(16384, C, 3, 5, seed=10 + k)
        got = evaluator.evaluate_population(pop, TrendParams())
        mode = evaluator.index_stats()["mode"]
        if mode == "full":
            np.testing.assert_array_equal(got, oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False))
            break
    assert mode == "full", evaluator.index_stats()
    np.testing.assert_array_equal(evaluator.evaluate_population(pop0, TrendParams()), want0)
    evaluator.upload(m)
    evaluator.prepare(0.03)
    np.testing.assert_array_equal(evaluator.evaluate_population(pop0, TrendParams()), want0)
    assert evaluator.index_stats()["mode"] == "full"


def test_auto_long_vectors_over_budget_use_lazy(evaluator):
    """Long pair vectors whose full index exceeds the budget (BASELINE config
    4's situation, scaled down): AUTO serves them from the lazy index, not the
    slab kernels, and keeps only the population's pairs."""
    R, C = 50000, 300  # full index 300^2 x 1664 words = 599 MB
    m = _matrix(R, C, 23)
    evaluator.upload(m)
    evaluator.set_table_budget(256 << 20)
    try:
        for k in range(3):
            pop = synth.random_population(3000, C, 3, 5, seed=50 + k % 2)
            for approx, neg in ((0.03, False), (0.03, True)):
                want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
                np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, neg)), want)
            st = evaluator.index_stats()
            assert st["mode"] == "lazy" and st["full_bytes"] == 0, st
        rows = evaluator.supporting_rows(pop.sequence(0), TrendParams(0.03, True))
        np.testing.assert_array_equal(rows, oracle.supporting_rows(m, pop.sequence(0), 0.03, True))
        assert evaluator.index_stats()["lazy_bytes"] <= 256 << 20
    finally:
        evaluator.set_table_budget(0)


def test_lazy_build_mode_is_validated(evaluator):
    """ebic_ctx_set_lazy_build takes 0 (auto), 1 (inline) or 2 (build first);
    anything else is an argument error that leaves the mode unchanged."""
    from paper_2105_01196_b200 import EbicError

    for bad in (-1, 3, 99):
        with pytest.raises(EbicError):
            evaluator.set_lazy_build(bad)
    for ok in (2, 1, 0):
        evaluator.set_lazy_build(ok)


def test_cold_route_first_batch_then_steady(evaluator):
    """AUTO: the first batch of a fresh lazy index takes the build-first route,
    later batches of the same population find every pair in the pool; a new
    population again brings new pairs.  Exact throughout, f32 and with zeros
    (empty brackets) in the matrix."""
    R, C = 9000, 300
    m = _matrix(R, C, 23)
    m[::5, ::7] = 0.0
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_LAZY)
    try:
        pops = [_pop(C, 2000, seed=40 + k) for k in range(2)]
        for k in (0, 0, 1, 0, 1):
            pop = pops[k]
            for neg in (False, True):
                want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, neg)
                got = evaluator.evaluate_population(pop, TrendParams(0.03, neg))
                np.testing.assert_array_equal(got, want, err_msg=f"pop {k} neg {neg}")
        assert evaluator.index_stats()["lazy_slots_used"] > 0
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)


@pytest.mark.parametrize("R", [4000, 33000])
def test_build_first_wide_matrix(evaluator, R):
    """The build-first route on a matrix too wide for two slab-builder CTAs per
    SM (1800 columns: the 1024-thread variant), short and long vectors,
    forward and reversed pairs, counts and row masks."""
    C = 1800
    m = _matrix(R, C, 29)
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_LAZY)
    evaluator.set_lazy_build(2)
    try:
        pop = _pop(C, 600, seed=7)
        for approx, neg in ((0.03, False), (0.0, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx, neg))
            np.testing.assert_array_equal(got, want, err_msg=f"R={R} approx={approx} neg={neg}")
        for j in (0, 3):
            rows = evaluator.supporting_rows(pop.sequence(j), TrendParams(0.03, True))
            np.testing.assert_array_equal(rows, oracle.supporting_rows(m, pop.sequence(j), 0.03, True))
    finally:
        evaluator.set_lazy_build(0)
        evaluator.set_path(EBIC_PATH_AUTO)
