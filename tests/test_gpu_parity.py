"""Parity of the CUDA path (through the C ABI) with the reference / the pinned oracle.

Bar: bit-exact integer counts and identical ascending row lists.
"""
import numpy as np
import pytest

import oracle
from conftest import golden_cases, load_golden
from paper_2105_01196_b200 import (EBIC_STORE_AUTO, EBIC_STORE_F32, EBIC_STORE_F64, EbicError, Population,
                                   TrendParams)
from paper_2105_01196_b200 import synth
from paper_2105_01196_b200._lib import (EBIC_PATH_AUTO, EBIC_PATH_PLANE, EBIC_PATH_PLANE_U32, EBIC_PATH_TABLE,
                                        EBIC_PATH_VALUE)

pytestmark = pytest.mark.gpu


@pytest.fixture(params=[EBIC_PATH_AUTO, EBIC_PATH_PLANE, EBIC_PATH_PLANE_U32, EBIC_PATH_VALUE],
                ids=["table", "plane", "plane_u32", "value"])
def path_evaluator(evaluator, request):
    """The same checks on every exact evaluation path: the default (the
    pair-trend index where it fits), the rank-plane slab kernels (packed 16-bit
    rank pairs where the slab fits), the 32-bit-word plane kernel, and the
    float value kernel."""
    evaluator.set_path(request.param)
    yield evaluator
    evaluator.set_path(EBIC_PATH_AUTO)


def _tp(s):
    return TrendParams(approx=s["approx"], negative_trends=s["negative"])


@pytest.mark.parametrize("name", golden_cases())
@pytest.mark.parametrize("store", [EBIC_STORE_AUTO, EBIC_STORE_F64])
def test_counts_and_rows_match_reference_golden(path_evaluator, name, store):
    evaluator = path_evaluator
    z, settings = load_golden(name)
    m = z["matrix"]
    chosen = evaluator.upload(m, store=store)
    exact = np.array_equal(m.astype(np.float32).astype(np.float64), m)
    assert chosen == (EBIC_STORE_F32 if (exact and store == EBIC_STORE_AUTO) else EBIC_STORE_F64)
    pop = Population(z["cols"], z["offsets"])
    for k, s in enumerate(settings):
        counts = evaluator.evaluate_population(pop, _tp(s))
        np.testing.assert_array_equal(counts, z[f"counts_{k}"], err_msg=f"{name} {s}")
        idx = z[f"rows_idx_{k}"]
        ro = z[f"rows_offsets_{k}"]
        batch = evaluator.supporting_rows_batch(Population.from_sequences([pop.sequence(i) for i in idx]), _tp(s))
        for j, i in enumerate(idx):
            want = z[f"rows_{k}"][ro[j]:ro[j + 1]]
            np.testing.assert_array_equal(batch[j], want)
            np.testing.assert_array_equal(evaluator.supporting_rows(pop.sequence(i), _tp(s)), want)


def test_row_supports_hand_vectors(evaluator):
    # test_trend.cpp:60-81
    def rs(rows, seq, approx, neg=False):
        evaluator.upload(np.array(rows, dtype=np.float64))
        return evaluator.row_supports(0, seq, TrendParams(approx=approx, negative_trends=neg))

    assert rs([[1.0, 2.0, 3.0]], [0, 1, 2], 0.0)
    assert not rs([[1.0, 2.0, 3.0]], [2, 1, 0], 0.0)
    assert rs([[3.0, 1.0, 2.0]], [1, 2, 0], 0.0)
    assert not rs([[1.0, 1.0]], [0, 1], 0.0)
    assert rs([[1.0, 1.0]], [0, 1], 0.05)
    assert not rs([[2.0, 2.0, 2.0]], [0, 1, 2], 0.0, True)


def _random_case(rng, R, Cn, f32=True, max_len=12):
    m = rng.standard_normal((R, Cn))
    if f32:
        m = m.astype(np.float32).astype(np.float64)
    m[rng.random(m.shape) < 0.03] = 0.0
    seqs = [rng.choice(Cn, size=int(rng.integers(1, min(Cn, max_len) + 1)), replace=False) for _ in range(300)]
    return m, Population.from_sequences(seqs)


@pytest.mark.parametrize("R", [1, 31, 256, 257, 1000, 4097])
@pytest.mark.parametrize("f32", [True, False])
def test_random_shapes_vs_oracle(path_evaluator, R, f32):
    evaluator = path_evaluator
    rng = np.random.default_rng(R * 7 + f32)
    m, pop = _random_case(rng, R, 40, f32)
    evaluator.upload(m)
    for approx in (0.0, 0.03, float(rng.uniform(0, 0.5)), 0.999):
        for neg in (False, True):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
            np.testing.assert_array_equal(got, want, err_msg=f"R={R} approx={approx} neg={neg}")


def _near_threshold_matrix(rng, R, Cn, approx):
    """Rows where each next value sits within a few float32 ulps of the reference
    threshold RN64(prev - RN64(approx*|prev|)) -- every pair lands in the float32
    filter's uncertain band and must be resolved by the exact double path."""
    m = np.empty((R, Cn), dtype=np.float64)
    x = rng.standard_normal(R).astype(np.float32)
    m[:, 0] = x
    for c in range(1, Cn):
        prev = m[:, c - 1]
        thr = prev - approx * np.abs(prev)
        t32 = thr.astype(np.float32)
        jitter = rng.integers(-2, 3, size=R)
        cur = t32.copy()
        for _ in range(2):
            cur = np.where(jitter > 0, np.nextafter(cur, np.float32(np.inf)), cur)
            cur = np.where(jitter < 0, np.nextafter(cur, np.float32(-np.inf)), cur)
            jitter = jitter - np.sign(jitter)
        m[:, c] = cur.astype(np.float64)
    return m


@pytest.mark.parametrize("approx", [0.03, 0.1, 0.5, 2**-20])
def test_filter_uncertain_band_is_exact(path_evaluator, approx):
    evaluator = path_evaluator
    rng = np.random.default_rng(11)
    m = _near_threshold_matrix(rng, 3000, 12, approx)
    assert np.array_equal(m.astype(np.float32).astype(np.float64), m)
    assert evaluator.upload(m) == EBIC_STORE_F32
    seqs = [list(range(a, b)) for a in range(0, 6) for b in range(a + 2, 13)]
    seqs += [list(range(b - 1, a - 1, -1)) for a in range(0, 6) for b in range(a + 2, 13)]
    pop = Population.from_sequences(seqs)
    for neg in (False, True):
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
        got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
        np.testing.assert_array_equal(got, want)
        assert want.sum() > 0


def test_subnormal_and_huge_values(path_evaluator):
    evaluator = path_evaluator
    rng = np.random.default_rng(5)
    vals = np.array([0.0, -0.0, 1e-45, -1e-45, 1.2e-38, -1.2e-38, 3.4e38, -3.4e38, 1.0, -1.0, 5e-40, -5e-40],
                    dtype=np.float32).astype(np.float64)
    m = rng.choice(vals, size=(2000, 12))
    assert evaluator.upload(m) == EBIC_STORE_F32
    seqs = [rng.choice(12, size=int(rng.integers(2, 7)), replace=False) for _ in range(500)]
    pop = Population.from_sequences(seqs)
    for approx in (0.0, 0.03, 0.999, 1e-8):
        for neg in (False, True):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
            np.testing.assert_array_equal(got, want)


def test_long_sequences_cross_smem_chunks(path_evaluator):
    evaluator = path_evaluator
    rng = np.random.default_rng(9)
    m = rng.standard_normal((5000, 300)).astype(np.float32)
    # sorted rows make long trends survive, so the column loop runs past the 64-index SMEM chunk
    m[:2500] = np.sort(m[:2500], axis=1)
    evaluator.upload(m)
    seqs = [np.sort(rng.choice(300, size=L, replace=False)) for L in (63, 64, 65, 128, 129, 200, 300)]
    seqs += [s[::-1] for s in seqs]
    pop = Population.from_sequences(seqs)
    for approx, neg in ((0.0, False), (0.03, True), (0.0, True)):
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
        got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
        np.testing.assert_array_equal(got, want)
        assert want.max() >= 2500


def _config_matrix(rows, cols, bic_rows, bic_cols, seed=1):
    if oracle.reference_available():
        # the reference generator (datagen.cpp:208-264), float32-quantised
        return oracle.ref_gen_scenario(rows, cols, bic_rows, bic_cols, 3, seed=seed, quantize=True)
    m, _ = synth.planted_trend_matrix(rows, cols, 3, bic_rows, bic_cols, seed=seed)
    return m


def test_config2_bit_exact(path_evaluator):
    evaluator = path_evaluator
    """BASELINE config 2: 10k x 500, P=4096, bit-exact counts vs the CPU oracle."""
    m = _config_matrix(10_000, 500, 500, 20)
    if oracle.reference_available():
        cols, offs = oracle.ref_init_population(4096, 500, seed=42)
        pop = Population(cols, offs)
    else:
        pop = synth.random_population(4096, 500, seed=42)
    assert evaluator.upload(m) == EBIC_STORE_F32
    for approx in (0.0, 0.03):
        for neg in (False, True):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
            np.testing.assert_array_equal(got, want)


def test_config3_full_size_bit_exact(evaluator):
    """BASELINE config 3 at full size on one GPU: 20k x 1000, P=16384."""
    m, _ = synth.planted_trend_matrix(20_000, 1000, 3, 500, 20, seed=3)
    pop = synth.random_population(16384, 1000, seed=42)
    evaluator.upload(m)
    tp = TrendParams(approx=0.03)
    want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False)
    np.testing.assert_array_equal(evaluator.evaluate_population(pop, tp), want)


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("policy", ["auto", "full", "lazy"])
def test_config3_full_size_vs_reference_library(evaluator, policy):
    """BASELINE config 3 at full size against the LIVE reference: the
    unmodified evaluate_population (oracle/_ref, trend.cpp:56-72) on a
    WorkerPool of all host cores, the whole 16384-candidate population, with
    the default policy (lazy index on a fresh matrix), the full index, and the
    lazy index; approx 0.03 and, with negatives, approx 0."""
    from paper_2105_01196_b200._lib import EBIC_PATH_LAZY, EBIC_PATH_TABLE

    m, _ = synth.planted_trend_matrix(20_000, 1000, 3, 500, 20, seed=3)
    pop = synth.random_population(16384, 1000, seed=42)
    evaluator.upload(m)
    evaluator.set_path({"auto": EBIC_PATH_AUTO, "full": EBIC_PATH_TABLE, "lazy": EBIC_PATH_LAZY}[policy])
    try:
        mat, rp, pool = oracle.RefMatrix(m.astype(np.float64)), oracle.RefPopulation(pop.cols, pop.offsets), oracle.RefPool(0)
        for approx, neg in ((0.03, False), (0.0, True)):
            want = oracle.ref_evaluate(mat, rp, approx, neg, pool)
            np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, neg)), want)
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)


@pytest.mark.skipif(not oracle.reference_available(), reason="oracle/_ref not built")
def test_config4_sample_vs_reference_library(evaluator):
    """BASELINE config 4 (200k x 2000, 1.6 GB f32): a 2048-candidate sample of
    the P=32768 population against the live reference library on all host
    cores (the whole population would take minutes of CPU)."""
    rng = np.random.default_rng(44)
    m = rng.standard_normal((200_000, 2000), dtype=np.float32)
    m[:4000] = np.sort(m[:4000], axis=1)  # rows that support long sorted candidates
    evaluator.upload(m)
    pop = synth.random_population(32768, 2000, seed=42)
    got = evaluator.evaluate_population(pop, TrendParams(approx=0.03))
    sample = np.sort(rng.choice(32768, size=2048, replace=False))
    sub = Population.from_sequences([pop.sequence(i) for i in sample])
    mat = oracle.RefMatrix(m.astype(np.float64))
    want = oracle.ref_evaluate(mat, oracle.RefPopulation(sub.cols, sub.offsets), 0.03, False, oracle.RefPool(0))
    np.testing.assert_array_equal(got[sample], want)
    del mat


def test_config4_full_size_properties(evaluator):
    """BASELINE config 4 (200k x 2000, 1.6 GB f32, P=32768): bit-exact on a candidate
    sample, plus size-independent properties over the whole population."""
    rng = np.random.default_rng(4)
    m = rng.standard_normal((200_000, 2000), dtype=np.float32)
    evaluator.upload(m)
    pop = synth.random_population(32768, 2000, seed=42)
    tp = TrendParams(approx=0.03)
    base = evaluator.evaluate_population(pop, tp)
    neg = evaluator.evaluate_population(pop, TrendParams(approx=0.03, negative_trends=True))
    loose = evaluator.evaluate_population(pop, TrendParams(approx=0.2))
    strict = evaluator.evaluate_population(pop, TrendParams(approx=0.0))
    assert (neg >= base).all() and (loose >= base).all() and (base >= strict).all()
    sample = rng.choice(32768, size=96, replace=False)
    sub = Population.from_sequences([pop.sequence(i) for i in sample])
    want = oracle.evaluate_population(m, sub.cols, sub.offsets, 0.03, False)
    np.testing.assert_array_equal(base[sample], want)
    # row-shard additivity: two shards summed == whole (the row-sharded exchange)
    half = 100_000
    evaluator.upload(m[:half], row_base=0)
    a = evaluator.evaluate_population(pop, tp)
    evaluator.upload(m[half:], row_base=half)
    b = evaluator.evaluate_population(pop, tp)
    np.testing.assert_array_equal(a + b, base)


@pytest.mark.parametrize("R", [1024, 65536, 1_000_000])
def test_microbench_shapes(path_evaluator, R):
    evaluator = path_evaluator
    rng = np.random.default_rng(R)
    m = rng.standard_normal((R, 64), dtype=np.float32)
    evaluator.upload(m)
    for L in (2, 16, 50):
        pop = synth.exact_len_population(64 if R > 100_000 else 256, 64, L, seed=L)
        for approx in (0.0, 0.03):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, False)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx))
            np.testing.assert_array_equal(got, want)


def test_support_rows_are_global_and_ascending(evaluator):
    rng = np.random.default_rng(2)
    m = rng.standard_normal((6000, 20)).astype(np.float32)
    seqs = [rng.choice(20, size=3, replace=False) for _ in range(20)]
    tp = TrendParams(approx=0.03, negative_trends=True)
    full = [oracle.supporting_rows(m, s, 0.03, True) for s in seqs]
    evaluator.upload(m[2000:], row_base=2000)
    got = evaluator.supporting_rows_batch(seqs, tp)
    for s, g, f in zip(seqs, got, full):
        np.testing.assert_array_equal(g, f[f >= 2000])
        assert (np.diff(g.astype(np.int64)) > 0).all()
    assert evaluator.row_supports(2000 + 5, seqs[0], tp) == oracle.row_supports(m, 2005, seqs[0], 0.03, True)


def test_device_pointer_path_and_external_stream(evaluator):
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    m = rng.standard_normal((10_000, 100)).astype(np.float32)
    evaluator.upload(m)
    pop = synth.random_population(2000, 100, seed=1)
    want = evaluator.evaluate_population(pop)
    d_cols = torch.from_numpy(pop.cols.view(np.int32)).cuda()
    d_offs = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
    d_counts = torch.full((len(pop),), -1, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        evaluator.evaluate_population_device(d_cols.data_ptr(), d_offs.data_ptr(), len(pop), d_counts.data_ptr(),
                                             TrendParams(), stream=s.cuda_stream)
    s.synchronize()
    np.testing.assert_array_equal(d_counts.cpu().numpy().view(np.uint32), want)
    evaluator.set_stream(s.cuda_stream)
    np.testing.assert_array_equal(evaluator.evaluate_population(pop), want)
    evaluator.set_stream(None)
    # a bad column on the device path is detected on device and reported by sync()
    bad = d_cols.clone()
    bad[0] = 100
    evaluator.evaluate_population_device(bad.data_ptr(), d_offs.data_ptr(), len(pop), d_counts.data_ptr())
    with pytest.raises(EbicError):
        evaluator.sync()
    evaluator.sync()  # flag cleared


def test_marshaller_ring(evaluator):
    rng = np.random.default_rng(4)
    m = rng.standard_normal((4000, 50)).astype(np.float32)
    evaluator.upload(m)
    # growing sizes force the ring's pinned buffers to grow while earlier
    # submissions are still in flight; more submissions than EBIC_MARSHAL_SLOTS
    sizes = [300, 700, 1500, 1400, 3000, 6000, 200, 9000, 50]
    pops = [synth.random_population(n, 50, seed=i) for i, n in enumerate(sizes)]
    outs = [np.zeros(len(p), dtype=np.uint32) for p in pops]
    tickets = [evaluator.submit(p, o) for p, o in zip(pops, outs)]
    for t in tickets:
        evaluator.wait(t)
    for p, o in zip(pops, outs):
        np.testing.assert_array_equal(o, oracle.evaluate_population(m, p.cols, p.offsets, 0.03, False))
    # a bad column in an early submission is reported by ITS wait, not by a later submit
    bad = Population(np.array([0, 99], np.uint32), np.array([0, 2], np.uint32))
    ob = np.zeros(1, dtype=np.uint32)
    tb = evaluator.submit(bad, ob)
    later = [evaluator.submit(p, o) for p, o in zip(pops[:5], outs[:5])]
    for t in later:
        evaluator.wait(t)
    with pytest.raises(EbicError, match="out of range"):
        evaluator.wait(tb)
    evaluator.wait(tb)  # reported once


def test_errors_are_reported_not_undefined(evaluator):
    m = np.random.default_rng(0).standard_normal((100, 10))
    evaluator.upload(m)
    with pytest.raises(EbicError, match="out of range"):
        evaluator.evaluate_population([[0, 10]])
    with pytest.raises(EbicError, match="empty"):
        evaluator.evaluate_population(Population(np.array([1], np.uint32), np.array([0, 0, 1], np.uint32)))
    with pytest.raises(EbicError, match="finite"):
        evaluator.evaluate_population([[0, 1]], TrendParams(approx=float("nan")))
    bad = m.copy()
    bad[3, 3] = np.inf
    with pytest.raises(EbicError, match="non-finite"):
        evaluator.upload(bad)
    with pytest.raises(EbicError) as ei:
        evaluator.upload(m, store=EBIC_STORE_F32)
    assert ei.value.status == 5
    # the failed uploads left no matrix behind
    with pytest.raises(EbicError) as ei:
        evaluator.evaluate_population([[0, 1]])
    assert ei.value.status == 3


def test_launches_are_counted(evaluator):
    m = np.random.default_rng(0).standard_normal((1000, 10)).astype(np.float32)
    evaluator.upload(m)
    evaluator.prepare(0.03)  # builds the rank plane for approx 0.03 (one launch)
    n0 = evaluator.launch_count()
    evaluator.evaluate_population([[0, 1, 2]] * 10)
    assert evaluator.launch_count() == n0 + 1
    evaluator.set_path(EBIC_PATH_VALUE)
    evaluator.evaluate_population([[0, 1, 2]] * 10)
    assert evaluator.launch_count() == n0 + 2
    evaluator.set_path(EBIC_PATH_AUTO)


def test_plane_is_rebuilt_per_approx_and_matrix(evaluator):
    rng = np.random.default_rng(8)
    m = rng.standard_normal((3000, 30)).astype(np.float32)
    pop = synth.random_population(500, 30, seed=3)
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_PLANE)
    try:
        for approx in (0.03, 0.0, 0.03, 0.5):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, True)
            np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, True)), want)
        m2 = m[::-1].copy()
        evaluator.upload(m2)
        want = oracle.evaluate_population(m2, pop.cols, pop.offsets, 0.5, True)
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(0.5, True)), want)
        # wider than the plane's column limit -> PLANE is refused, AUTO falls back to the value kernel
        wide = rng.standard_normal((64, 9000)).astype(np.float32)
        evaluator.upload(wide)
        with pytest.raises(EbicError):
            evaluator.evaluate_population([[0, 1, 8999]])
        evaluator.set_path(EBIC_PATH_AUTO)
        want = oracle.evaluate_population(wide, np.array([0, 1, 8999], np.uint32), np.array([0, 3], np.uint32), 0.03,
                                          False)
        np.testing.assert_array_equal(evaluator.evaluate_population([[0, 1, 8999]]), want)
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)


@pytest.mark.parametrize("n_cols", [600, 1000, 1024, 1100, 2048, 3000, 5000])
def test_wide_matrices_every_slab_variant(path_evaluator, n_cols):
    """Column counts that select each slab layout: packed rank pairs with two
    (C <= 1024) and four (C <= 2048) candidates per warp instruction, and
    32-bit plane words with 16- and 8-row slabs above that."""
    evaluator = path_evaluator
    rng = np.random.default_rng(n_cols)
    R = 1500
    m = rng.standard_normal((R, n_cols)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)  # long trends survive
    m[rng.random(m.shape) < 0.01] = 0.0
    seqs = [rng.choice(n_cols, size=int(rng.integers(1, 13)), replace=False) for _ in range(700)]
    seqs += [np.sort(rng.choice(n_cols, size=L, replace=False)) for L in (8, 9, 20, 40)]
    pop = Population.from_sequences(seqs)
    evaluator.upload(m)
    for approx, neg in ((0.03, False), (0.0, True), (0.2, True)):
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
        got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
        np.testing.assert_array_equal(got, want, err_msg=f"C={n_cols} approx={approx} neg={neg}")


@pytest.mark.parametrize("n_cols", [2, 33, 64, 65, 200, 511, 1000, 1024, 2000, 3000])
@pytest.mark.parametrize("f64", [False, True])
def test_plane_builders_agree(n_cols, f64, monkeypatch):
    """The row-tile plane builder (register or warp shared-memory sort) and the
    per-row block-sort builder give identical counts -- on rows full of ties,
    signed zeros, subnormals and huge values, for f32 and f64 stores."""
    from paper_2105_01196_b200 import Evaluator

    rng = np.random.default_rng(n_cols)
    vals = np.array([0.0, -0.0, 1e-45, -1e-45, 1.0, 1.0, -1.0, 3.4e38, -3.4e38, 0.97, 1.03], dtype=np.float32)
    m = np.where(rng.random((777, n_cols)) < 0.5, rng.choice(vals, size=(777, n_cols)),
                 rng.standard_normal((777, n_cols)).astype(np.float32)).astype(np.float64)
    if f64:
        m = m + rng.standard_normal(m.shape) * 1e-9  # not float32-representable: f64 store
    seqs = [rng.choice(n_cols, size=int(rng.integers(1, min(n_cols, 7) + 1)), replace=False) for _ in range(400)]
    pop = Population.from_sequences(seqs)
    settings = ((0.0, True), (0.03, False), (0.5, True))
    results = []
    for builder in ("2", "1"):
        monkeypatch.setenv("EBIC_PLANE_BUILDER", builder)
        with Evaluator(0) as ev:
            assert ev.upload(m) == (EBIC_STORE_F64 if f64 else EBIC_STORE_F32)
            ev.set_path(EBIC_PATH_PLANE)
            results.append([ev.evaluate_population(pop, TrendParams(a, neg)) for a, neg in settings])
    for got_tile, got_block, (a, neg) in zip(results[0], results[1], settings):
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, a, neg)
        np.testing.assert_array_equal(got_tile, want)
        np.testing.assert_array_equal(got_block, want)


PAIR_LAYOUTS = [(2, 1), (2, 2), (2, 4), (1, 1), (1, 2), (1, 4)]


@pytest.mark.gpu
@pytest.mark.parametrize("layout", PAIR_LAYOUTS, ids=[f"p{p}s{s}" for p, s in PAIR_LAYOUTS])
@pytest.mark.parametrize("n_cols", [40, 250, 500, 1000, 2000])
def test_every_pair_layout(evaluator, layout, n_cols):
    """Each packed-pair layout of the hot kernel (row pairs per lane x
    candidates per warp instruction), forced, against the C oracle: short and
    long candidates (record tail from the CSR), negatives, ragged last slab.
    Layouts whose slab does not fit run on the 32-bit-word kernel instead."""
    rng = np.random.default_rng(1000 + n_cols)
    R = 1000 + 37
    m = rng.standard_normal((R, n_cols)).astype(np.float32)
    m[: R // 4] = np.sort(m[: R // 4], axis=1)
    m[R // 4: R // 2] = -np.sort(m[R // 4: R // 2], axis=1)
    m[rng.random(m.shape) < 0.02] = 0.0
    seqs = [rng.choice(n_cols, size=int(rng.integers(1, 11)), replace=False) for _ in range(900)]
    seqs += [np.sort(rng.choice(n_cols, size=min(L, n_cols), replace=False)) for L in (8, 12, 30)]
    pop = Population.from_sequences(seqs)
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_PLANE)
    evaluator.set_pair_layout(*layout)
    try:
        for approx, neg in ((0.03, False), (0.0, True), (0.3, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
            np.testing.assert_array_equal(got, want, err_msg=f"C={n_cols} layout={layout} approx={approx} neg={neg}")
    finally:
        evaluator.set_pair_layout(0, 0)
        evaluator.set_path(EBIC_PATH_AUTO)


def _pinned_u32(a):
    import torch

    t = torch.empty(max(a.size, 1), dtype=torch.int32, pin_memory=True)
    v = t.numpy().view(np.uint32)[: a.size]
    v[:] = a
    return t, v


@pytest.mark.parametrize("layout", ["separate", "one_block"])
@pytest.mark.parametrize("path", [EBIC_PATH_AUTO, EBIC_PATH_PLANE_U32, EBIC_PATH_VALUE], ids=["pair", "u32", "value"])
def test_zero_copy_host_path(evaluator, layout, path):
    """Page-locked host arrays: inputs DMA'd directly (one copy for an
    [offsets | cols] block), counts written by the kernel straight into the
    page-locked output (pair kernel) or copied back (other kernels); a bad
    column is reported and the next call is clean."""
    rng = np.random.default_rng(77)
    m = rng.standard_normal((3000, 700)).astype(np.float32)
    m[:500] = np.sort(m[:500], axis=1)
    pop = Population.from_sequences(rng.choice(700, size=int(rng.integers(2, 10)), replace=False)
                                    for _ in range(5000))
    evaluator.upload(m)
    evaluator.set_path(path)
    keep = []
    try:
        if layout == "one_block":
            t, buf = _pinned_u32(np.concatenate([pop.offsets, pop.cols]))
            keep.append(t)
            ppop = Population(buf[pop.offsets.size:], buf[: pop.offsets.size])
        else:
            (t1, c), (t2, o) = _pinned_u32(pop.cols), _pinned_u32(pop.offsets)
            keep += [t1, t2]
            ppop = Population(c, o)
        t3, out = _pinned_u32(np.full(len(pop), 0xDEADBEEF, np.uint32))
        keep.append(t3)
        for approx, neg in ((0.03, False), (0.0, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(ppop, TrendParams(approx=approx, negative_trends=neg), out=out)
            np.testing.assert_array_equal(got, want)
        # a bad column: reported, and the following call is clean again
        bad = ppop.cols.copy()
        bad_pop = Population(bad, ppop.offsets.copy())
        bad[3] = 700
        t4, bc = _pinned_u32(bad)
        keep.append(t4)
        with pytest.raises(EbicError):
            evaluator.evaluate_population(Population(bc, ppop.offsets), TrendParams(), out=out)
        del bad_pop
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False)
        np.testing.assert_array_equal(evaluator.evaluate_population(ppop, TrendParams(), out=out), want)
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)



@pytest.mark.parametrize("zc_read_max", ["0", "1000000000"])
@pytest.mark.parametrize("R", [500, 20000, 40000])
def test_small_batches_read_in_place(monkeypatch, zc_read_max, R):
    """Page-locked populations small enough (EBIC_ZC_READ_MAX) are read in
    place by the index kernel over the bus instead of being DMA'd: the same
    counts either way, on the lane-group, TMA and lazy long-vector kernels,
    including a bad candidate's error and the clean call after it."""
    from paper_2105_01196_b200 import Evaluator

    monkeypatch.setenv("EBIC_ZC_READ_MAX", zc_read_max)  # read at context creation
    rng = np.random.default_rng(R)
    m = rng.standard_normal((R, 250)).astype(np.float32)
    m[: R // 4] = np.sort(m[: R // 4], axis=1)
    pop = Population.from_sequences(rng.choice(250, size=int(rng.integers(1, 7)), replace=False) for _ in range(392))
    with Evaluator(0) as ev:
        ev.upload(m)
        keep = []
        t, buf = _pinned_u32(np.concatenate([pop.offsets, pop.cols]))
        keep.append(t)
        ppop = Population(buf[pop.offsets.size:], buf[: pop.offsets.size])
        t2, out = _pinned_u32(np.full(len(pop), 0xDEADBEEF, np.uint32))
        keep.append(t2)
        for approx, neg in ((0.03, False), (0.0, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            for _ in range(2):  # (the lazy index: built on the first call, read on the second)
                got = ev.evaluate_population(ppop, TrendParams(approx=approx, negative_trends=neg), out=out)
                np.testing.assert_array_equal(got, want)
        bad = ppop.cols.copy()
        bad[2] = 250
        t3, bc = _pinned_u32(bad)
        keep.append(t3)
        with pytest.raises(EbicError):
            ev.evaluate_population(Population(bc, ppop.offsets), TrendParams(), out=out)
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False)
        np.testing.assert_array_equal(ev.evaluate_population(ppop, TrendParams(), out=out), want)


@pytest.mark.parametrize("R", [1, 31, 32, 33, 127, 1000, 1037, 4099, 4129, 10000, 20000, 32768, 32800])
@pytest.mark.parametrize("n_cols", [2, 37, 300])
def test_pair_trend_index_vs_oracle(evaluator, R, n_cols):
    """The pair-trend index (forced) against the C oracle: ragged row counts
    (partial words and pair vectors), tiny and mid widths, duplicate columns,
    length-1 and long candidates, negatives, several approx values; row masks
    (supporting_rows) from the same index."""
    rng = np.random.default_rng(R * 1000 + n_cols)
    m = rng.standard_normal((R, n_cols)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)
    m[rng.random(m.shape) < 0.05] = 0.0
    seqs = [rng.choice(n_cols, size=int(rng.integers(1, min(n_cols, 9) + 1)), replace=False) for _ in range(600)]
    seqs += [rng.integers(0, n_cols, size=int(rng.integers(2, 6))) for _ in range(50)]  # duplicates allowed
    seqs += [np.sort(rng.choice(n_cols, size=min(n_cols, 40), replace=False))]
    pop = Population.from_sequences(seqs)
    evaluator.upload(m)
    evaluator.set_path(EBIC_PATH_TABLE)
    try:
        for approx, neg in ((0.03, False), (0.0, True), (0.25, True), (0.03, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            got = evaluator.evaluate_population(pop, TrendParams(approx=approx, negative_trends=neg))
            np.testing.assert_array_equal(got, want, err_msg=f"R={R} C={n_cols} approx={approx} neg={neg}")
        for j in (0, 7, len(pop) - 1):
            for approx, neg in ((0.03, False), (0.1, True)):
                rows = evaluator.supporting_rows(pop.sequence(j), TrendParams(approx, neg))
                np.testing.assert_array_equal(rows, oracle.supporting_rows(m, pop.sequence(j), approx, neg))
        assert evaluator.index_info()[1]
    finally:
        evaluator.set_path(EBIC_PATH_AUTO)


def test_pair_trend_index_budget_and_fallback(evaluator):
    """AUTO builds the full index only within the budget; below it the lazy
    index serves (same counts); the index is rebuilt per approx and per matrix."""
    rng = np.random.default_rng(5)
    m = rng.standard_normal((2000, 120)).astype(np.float32)
    pop = synth.random_population(800, 120, seed=9)
    evaluator.upload(m)
    need, built = evaluator.index_info()
    assert need == 120 * 120 * 64 * 4 and not built  # wp = round_up(ceil(2000/32), 4) = 64 words
    try:
        evaluator.set_table_budget(need - 1)
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False)
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams()), want)
        assert not evaluator.index_info()[1] and evaluator.index_stats()["mode"] == "lazy"
        evaluator.set_table_budget(1 << 40)
        for approx in (0.03, 0.2, 0.0, 0.03):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, True)
            np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, True)), want)
            assert evaluator.index_info()[1]
        m2 = m[:, ::-1].copy()
        evaluator.upload(m2)
        assert not evaluator.index_info()[1]
        want = oracle.evaluate_population(m2, pop.cols, pop.offsets, 0.03, False)
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams()), want)
    finally:
        evaluator.set_table_budget(0)  # the library default


@pytest.mark.parametrize("layout", ["separate", "one_block"])
def test_zero_copy_pipelined_pieces(evaluator, layout):
    """Large page-locked populations go over in pieces while earlier pieces are
    evaluated (index path): counts and errors as the single-shot path, for
    ragged piece boundaries and long candidates."""
    rng = np.random.default_rng(99)
    m = rng.standard_normal((5000, 300)).astype(np.float32)
    m[:800] = np.sort(m[:800], axis=1)
    seqs = [rng.choice(300, size=int(rng.integers(1, 12)), replace=False) for _ in range(9001)]
    seqs[4500] = np.sort(rng.choice(300, size=60, replace=False))
    pop = Population.from_sequences(seqs)
    evaluator.upload(m)
    keep = []
    if layout == "one_block":
        t, buf = _pinned_u32(np.concatenate([pop.offsets, pop.cols]))
        keep.append(t)
        ppop = Population(buf[pop.offsets.size:], buf[: pop.offsets.size])
    else:
        (t1, c), (t2, o) = _pinned_u32(pop.cols), _pinned_u32(pop.offsets)
        keep += [t1, t2]
        ppop = Population(c, o)
    t3, out = _pinned_u32(np.zeros(len(pop), np.uint32))
    keep.append(t3)
    for approx, neg in ((0.03, False), (0.1, True)):
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
        np.testing.assert_array_equal(evaluator.evaluate_population(ppop, TrendParams(approx, neg), out=out), want)
    assert evaluator.index_info()[1]
    # a bad column in the last piece and an empty candidate in the first
    bad = ppop.cols.copy()
    bad[-1] = 300
    tb, bc = _pinned_u32(bad)
    keep.append(tb)
    with pytest.raises(EbicError, match="out of range"):
        evaluator.evaluate_population(Population(bc, ppop.offsets), TrendParams(), out=out)
    offs = ppop.offsets.copy()
    offs[3] = offs[2]
    to, bo = _pinned_u32(offs)
    keep.append(to)
    with pytest.raises(EbicError, match="empty"):
        evaluator.evaluate_population(Population(ppop.cols, bo), TrendParams(), out=out)
    want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, False)
    np.testing.assert_array_equal(evaluator.evaluate_population(ppop, TrendParams(), out=out), want)


def test_load_tsv_into_device_store(evaluator, tmp_path):
    """ebic_matrix_load_tsv: the reference TSV format parsed on all host threads
    into page-locked memory and uploaded; counts identical to the reference
    evaluator on the reference parser's matrix."""
    if not oracle.ref_io_available():
        pytest.skip("reference io.cpp not built")
    m = synth.planted_trend_matrix(3000, 150, 2, 300, 10, seed=4)[0].astype(np.float64)
    m[5, 7] = 0.1  # not float32-exact: the store stays f64
    f = tmp_path / "m.tsv"
    oracle.ref_write_matrix_tsv(f, m)
    rows, cols, store = evaluator.load_tsv(f)
    assert (rows, cols, store) == (3000, 150, EBIC_STORE_F64)
    ref_m = oracle.ref_parse_matrix_tsv(f)
    pop = synth.random_population(2000, 150, seed=5)
    for approx, neg in ((0.03, False), (0.0, True)):
        want = oracle.evaluate_population(ref_m, pop.cols, pop.offsets, approx, neg)
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, neg)), want)


@pytest.mark.parametrize("neg", [False, True])
def test_pair_trend_index_long_vectors_many_candidates(neg):
    """Long pair vectors (40000 rows: 1280 words, 320 uint4 slices) and enough
    candidates to select the multi-pass warp kernel; ragged last pass; vs the
    oracle.  Counts (twice), row masks, and a bad column (error)."""
    from paper_2105_01196_b200 import Evaluator
    ev = Evaluator(0)
    try:
        rng = np.random.default_rng(40)
        R, Cn = 40000, 16
        m = rng.standard_normal((R, Cn)).astype(np.float32)
        m[:9000] = np.sort(m[:9000], axis=1)
        seqs = [rng.choice(Cn, size=int(rng.integers(1, 7)), replace=False) for _ in range(5000)]
        pop = Population.from_sequences(seqs)
        ev.upload(m)
        ev.set_path(EBIC_PATH_TABLE)
        for approx in (0.03, 0.0, 0.03):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            np.testing.assert_array_equal(ev.evaluate_population(pop, TrendParams(approx, neg)), want)
        rows = ev.supporting_rows_batch(pop, TrendParams(0.03, neg))
        for j in (0, 1, 2, 4999):
            np.testing.assert_array_equal(rows[j], oracle.supporting_rows(m, seqs[j], 0.03, neg))
        bad = seqs[:4900] + [[0, Cn]] + seqs[4900:]
        with pytest.raises(EbicError):
            ev.evaluate_population(bad, TrendParams(0.03, neg))
        want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, neg)
        np.testing.assert_array_equal(ev.evaluate_population(pop, TrendParams(0.03, neg)), want)
    finally:
        ev.close()


def _overlap_want(m, seqs, approx, neg):
    rows = [oracle.supporting_rows(m, s, approx, neg) for s in seqs]
    n = len(seqs)
    inter = np.zeros((n, n), dtype=np.uint64)
    for i in range(n):
        for j in range(n):
            inter[i, j] = np.intersect1d(rows[i], rows[j], assume_unique=True).size
    return np.array([r.size for r in rows], dtype=np.uint64), inter


@pytest.mark.parametrize("R", [1, 33, 1000, 4099])
@pytest.mark.parametrize("neg", [False, True])
def test_support_overlaps_vs_oracle(path_evaluator, R, neg):
    """ebic_support_overlap_batch: sizes and pairwise |rows_i n rows_j| equal the
    reference row lists' intersections (evolution.cpp:44-51's counts), on every
    path; duplicates in the batch, single-column candidates (all rows), and
    sizes straddling the overlap kernel's 8-candidate tiles."""
    rng = np.random.default_rng(R)
    m = rng.standard_normal((R, 40)).astype(np.float32).astype(np.float64)
    m[:, 5] = m[:, 4]  # ties
    seqs = [list(rng.choice(40, size=int(rng.integers(2, 7)), replace=False)) for _ in range(17)]
    seqs += [seqs[3], [7], [4, 5], [5, 4]]
    path_evaluator.upload(m)
    approx = 0.03
    sizes, inter = path_evaluator.support_overlaps(seqs, TrendParams(approx=approx, negative_trends=neg))
    ws, wi = _overlap_want(m, seqs, approx, neg)
    np.testing.assert_array_equal(sizes, ws)
    np.testing.assert_array_equal(inter, wi)
    counts = path_evaluator.evaluate_population(seqs, TrendParams(approx=approx, negative_trends=neg))
    np.testing.assert_array_equal(sizes, counts.astype(np.uint64))


def test_support_overlaps_edges(evaluator):
    rng = np.random.default_rng(5)
    m = rng.standard_normal((500, 20)).astype(np.float32)
    evaluator.upload(m)
    s, i = evaluator.support_overlaps([])
    assert s.size == 0 and i.size == 0
    with pytest.raises(EbicError):
        evaluator.support_overlaps([[0, 99]])  # column out of range
    with pytest.raises(EbicError):
        evaluator.support_overlaps([[0, 1]] * 4097)  # over EBIC_OVERLAP_MAX
    # the largest batch: a symmetric matrix whose diagonal is the counts
    pop = synth.random_population(4096, 20, seed=2)
    sizes, inter = evaluator.support_overlaps(pop)
    np.testing.assert_array_equal(np.diag(inter), sizes)
    np.testing.assert_array_equal(inter, inter.T)
    np.testing.assert_array_equal(sizes, evaluator.evaluate_population(pop).astype(np.uint64))
    k = [0, 17, 4095]
    rows = evaluator.supporting_rows_batch(Population.from_sequences([pop.sequence(x) for x in k]))
    for a in range(3):
        for b in range(3):
            assert inter[k[a], k[b]] == np.intersect1d(rows[a], rows[b]).size


def test_upload_from_device_memory(evaluator):
    """ebic_matrix_upload_device_f32/_f64: a row-major matrix already in GPU
    memory (what an NCCL broadcast fills) builds the same store as the host
    upload -- f32, f64 that is f32-exact (f32 store), f64 that is not (f64
    store), a row shard with row_base -- and the counts and rows match the
    oracle; the source buffer is left unchanged; host pointers are refused."""
    import torch

    rng = np.random.default_rng(12)
    m32 = rng.standard_normal((3001, 60)).astype(np.float32)
    m32[:800] = np.sort(m32[:800], axis=1)
    pop = synth.random_population(3000, 60, seed=4)
    tp = TrendParams(approx=0.03, negative_trends=True)
    want = oracle.evaluate_population(m32.astype(np.float64), pop.cols, pop.offsets, 0.03, True)
    try:
        t = torch.from_numpy(m32).cuda()
        torch.cuda.synchronize()  # (the caller makes sure the buffer has landed)
        assert evaluator.upload_device(t.data_ptr(), 3001, 60, "f32") == EBIC_STORE_F32
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, tp), want)
        assert torch.equal(t.cpu(), torch.from_numpy(m32))
        t64 = torch.from_numpy(m32.astype(np.float64)).cuda()
        torch.cuda.synchronize()
        assert evaluator.upload_device(t64.data_ptr(), 3001, 60, "f64") == EBIC_STORE_F32
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, tp), want)
        m64 = m32.astype(np.float64) + 1e-12
        t64 = torch.from_numpy(m64).cuda()
        torch.cuda.synchronize()
        assert evaluator.upload_device(t64.data_ptr(), 3001, 60, "f64") == EBIC_STORE_F64
        np.testing.assert_array_equal(evaluator.evaluate_population(pop, tp),
                                      oracle.evaluate_population(m64, pop.cols, pop.offsets, 0.03, True))
        # a row shard: rows [1000, 3001) with global row ids
        sub = t[1000:]
        evaluator.upload_device(sub.data_ptr(), 2001, 60, "f32", row_base=1000)
        rows = evaluator.supporting_rows(pop.sequence(0), tp)
        full = oracle.supporting_rows(m32.astype(np.float64), pop.sequence(0), 0.03, True)
        np.testing.assert_array_equal(rows, full[full >= 1000])
        with pytest.raises(EbicError):
            evaluator.upload_device(m32.ctypes.data, 3001, 60, "f32")  # host memory
    finally:
        evaluator.upload(m32)


def test_index_allocation_kept_across_uploads(evaluator):
    """A new upload reuses the previous pair-trend index allocation when the
    new index fits it (same shape; smaller but at least half) and reallocates
    otherwise (larger; much smaller); the index is rebuilt for every matrix
    and the counts follow the current matrix."""
    rng = np.random.default_rng(21)
    for R, C in ((5000, 120), (5000, 120), (4000, 110), (9000, 150), (600, 30), (5000, 120)):
        m = rng.standard_normal((R, C)).astype(np.float32)
        m[: R // 4] = np.sort(m[: R // 4], axis=1)
        pop = synth.random_population(1500, C, seed=R + C)
        evaluator.upload(m)
        for approx, neg in ((0.03, False), (0.0, True)):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            np.testing.assert_array_equal(evaluator.evaluate_population(pop, TrendParams(approx, neg)), want)
        assert evaluator.index_info()[1]


@pytest.mark.parametrize("R", [5000, 20000, 70000])
@pytest.mark.parametrize("neg", [False, True])
def test_back_to_back_launches_programmatic_dependent(evaluator, R, neg):
    """Count kernels issued back to back on one stream overlap (programmatic
    dependent launch: kernel k+1 starts while kernel k drains).  Every launch's
    counts must still be exact, and a buffer written by several launches must
    hold the LAST one's counts (kernel k+1 waits for kernel k before storing)."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(R)
    m = rng.standard_normal((R, 300)).astype(np.float32)
    m[: R // 4] = np.sort(m[: R // 4], axis=1)
    evaluator.upload(m)
    tp = TrendParams(0.03, neg)
    pops = [synth.random_population(3000 + 500 * k, 300, 1 if k == 2 else 2, 7, seed=50 + k) for k in range(4)]
    want = [oracle.evaluate_population(m, p.cols, p.offsets, 0.03, neg) for p in pops]
    dev = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda())
           for p in pops]
    n_max = max(len(p) for p in pops)
    shared = torch.full((n_max,), -1, dtype=torch.int32, device="cuda")
    outs = [torch.full((len(pops[i % 4]),), -1, dtype=torch.int32, device="cuda") for i in range(24)]
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    for i in range(24):
        dc, do = dev[i % 4]
        n = len(pops[i % 4])
        evaluator.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, outs[i].data_ptr(), tp,
                                             stream=s.cuda_stream)
        evaluator.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, shared.data_ptr(), tp,
                                             stream=s.cuda_stream)
    s.synchronize()
    evaluator.sync()
    for i in range(24):
        np.testing.assert_array_equal(outs[i].cpu().numpy().view(np.uint32), want[i % 4], err_msg=f"launch {i}")
    last = want[23 % 4]
    got = shared.cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got[:len(last)], last)
    # positions past the last population were last written by a longer one
    longest = max(range(4), key=lambda k: (len(pops[k]), -k))
    np.testing.assert_array_equal(got[len(last):], want[longest][len(last):])
