"""Multi-process (world_size 2, gloo, CPU) coverage of the sharding layer.

The CUDA evaluator is replaced by an oracle-backed local evaluator with the same
interface (test infrastructure), so what is exercised here is exactly the
product's partitioning and exchange logic in paper_2105_01196_b200/shard.py:
row shards + all_reduce(SUM) of counts, population slices + all_gather, and
rank-ordered concatenation of ascending row lists.
"""
import os
import socket

import numpy as np
import pytest

from paper_2105_01196_b200.shard import ShardedEvaluator, pop_range, row_range, slice_population
from paper_2105_01196_b200.trend import Population, TrendParams


class OracleLocal:
    """Same interface as paper_2105_01196_b200.Evaluator, computed by the CPU oracle."""

    def upload(self, matrix, row_base=0, store=0):
        self.m = np.ascontiguousarray(matrix, dtype=np.float64)
        self.row_base = row_base

    def evaluate_population(self, pop, p):
        import oracle

        return oracle.evaluate_population(self.m, pop.cols, pop.offsets, p.approx, p.negative_trends, threads=1)

    def supporting_rows_batch(self, pop, p):
        import oracle

        return [oracle.supporting_rows(self.m, pop.sequence(i), p.approx, p.negative_trends) + self.row_base
                for i in range(len(pop))]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(0)
    m = rng.standard_normal((1001, 30)).astype(np.float32).astype(np.float64)
    m[:300] = np.sort(m[:300], axis=1)
    seqs = [rng.choice(30, size=int(rng.integers(2, 6)), replace=False) for _ in range(157)]
    return m, Population.from_sequences(seqs)


def _worker(rank, world, port, mode, q, source="local"):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, pop = _problem()
        given = m if (source == "local" or rank == 0) else None  # broadcast: only rank 0 has it
        sev = ShardedEvaluator(OracleLocal(), given, mode=mode, dist=dist, source=source)
        out = {}
        for approx, neg in ((0.03, False), (0.0, True)):
            tp = TrendParams(approx=approx, negative_trends=neg)
            out[(approx, neg)] = (sev.evaluate_population(pop, tp),
                                  sev.supporting_rows_batch(slice_population(pop, 0, 9), tp))
        q.put((rank, out, sev.spec.rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("source", ["local", "broadcast"])
@pytest.mark.parametrize("mode", ["rows", "pop"])
def test_world2_gloo_matches_single_process(mode, source):
    import torch.multiprocessing as mp

    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q, source)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, pop = _problem()
    shards = sorted(r[2] for r in results)
    if mode == "rows":
        assert shards == [(0, 501), (501, 1001)]
    for _, out, _ in results:
        for (approx, neg), (counts, rows) in out.items():
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            np.testing.assert_array_equal(counts, want)
            for i, r in enumerate(rows):
                np.testing.assert_array_equal(r, oracle.supporting_rows(m, pop.sequence(i), approx, neg))


def test_ranges_partition_exactly():
    for n in (0, 1, 7, 1000, 20001):
        for world in (1, 2, 3, 8):
            spans = [row_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
            assert [pop_range(n, r, world) for r in range(world)] == spans


def test_slice_population_rebases_offsets():
    pop = Population.from_sequences([[0, 1], [2, 3, 4], [5], [6, 7]])
    sub = slice_population(pop, 1, 3)
    assert sub.offsets.tolist() == [0, 3, 4]
    assert sub.cols.tolist() == [2, 3, 4, 5]
