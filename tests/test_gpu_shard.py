"""The sharded layer with the REAL CUDA evaluator: two ranks (gloo) sharing one
GPU, row-sharded and population-sharded, checked against the oracle.  (The
round's GPU box has one B200; NCCL refuses two ranks on one device, so the
collective here is gloo -- the exchange logic is the same code path.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(7)
    m = rng.standard_normal((5003, 300)).astype(np.float32)
    m[:1500] = np.sort(m[:1500], axis=1)
    from paper_2105_01196_b200 import synth

    pop = synth.random_population(3001, 300, 2, 9, seed=5)
    return m, pop


def _worker(rank, world, port, mode, q):
    import torch.distributed as dist

    from paper_2105_01196_b200 import Evaluator, TrendParams
    from paper_2105_01196_b200.shard import ShardedEvaluator, slice_population

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, pop = _problem()
        ev = Evaluator(0)
        sev = ShardedEvaluator(ev, m, mode=mode, dist=dist)
        out = {}
        for approx, neg in ((0.03, False), (0.0, True)):
            tp = TrendParams(approx=approx, negative_trends=neg)
            out[(approx, neg)] = (sev.evaluate_population(pop, tp),
                                  sev.supporting_rows_batch(slice_population(pop, 0, 12), tp))
        q.put((rank, out, sev.spec.rows, ev.launch_count()))
        ev.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["rows", "pop"])
def test_two_ranks_one_gpu_match_oracle(mode):
    import torch.multiprocessing as mp

    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m, pop = _problem()
    for _, out, _, launches in results:
        assert launches > 0  # the CUDA kernels ran
        for (approx, neg), (counts, rows) in out.items():
            np.testing.assert_array_equal(counts, oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg))
            for i, r in enumerate(rows):
                np.testing.assert_array_equal(r, oracle.supporting_rows(m, pop.sequence(i), approx, neg))
