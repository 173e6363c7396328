"""Row-sharded step with the count reduction over peer memory (ebic_xchg.cuh).

Every rank evaluates the whole population on its row block and the partial
counts are summed through exchange windows mapped into every rank.  Here the
ranks are contexts sharing one B200: in one process (windows mapped by device
pointer, kernels of the ranks running concurrently on their own streams), and
in two processes (windows mapped through CUDA IPC, handles exchanged with a
gloo all_gather).  The sums must equal the reference counts on the whole
matrix, bit for bit, over several epochs (both inbox parities)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2105_01196_b200 import EbicError, Evaluator, Population, TrendParams, build, synth
from paper_2105_01196_b200.shard import row_range

pytestmark = pytest.mark.gpu


def _matrix(R, C, seed):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((R, C)).astype(np.float32)
    m[: R // 3] = np.sort(m[: R // 3], axis=1)
    return m


@pytest.mark.parametrize("world", [2, 3])
def test_rows_sum_in_process(world):
    import torch

    build.build_ext()
    R, C = 2501, 90
    m = _matrix(R, C, world)
    evs = [Evaluator(0) for _ in range(world)]
    try:
        for g, ev in enumerate(evs):
            b, e = row_range(R, g, world)
            ev.upload(np.ascontiguousarray(m[b:e]), row_base=b)
            ev.prepare(0.03)  # index buffers allocated before any rank's exchange kernel spins
            ev.xchg_create(world, g, 5000)
        wins = [ev.xchg_window() for ev in evs]
        for ev in evs:
            ev.xchg_open_local(wins)
        streams = [torch.cuda.Stream() for _ in range(world)]
        for step in range(5):  # several epochs: both inbox parities, reused windows
            pop = synth.random_population(4000 + 100 * step, C, 2, 8, seed=step)
            approx, neg = ((0.03, False), (0.0, True), (0.2, True))[step % 3]
            d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
            d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
            outs = [torch.full((len(pop),), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
            for g, ev in enumerate(evs):  # all ranks in flight at once
                ev.evaluate_population_rows_sum_device(d_c.data_ptr(), d_o.data_ptr(), len(pop), outs[g].data_ptr(),
                                                       TrendParams(approx, neg), stream=streams[g].cuda_stream)
            for ev in evs:
                ev.sync()
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            for g in range(world):
                np.testing.assert_array_equal(outs[g].cpu().numpy().view(np.uint32), want,
                                              err_msg=f"rank {g} step {step}")
        with pytest.raises(EbicError):  # over the window's capacity
            pop = synth.random_population(6000, C, 2, 5, seed=9)
            d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
            d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
            out = torch.empty(6000, dtype=torch.int32, device="cuda")
            evs[0].evaluate_population_rows_sum_device(d_c.data_ptr(), d_o.data_ptr(), 6000, out.data_ptr())
    finally:
        for ev in evs:
            ev.close()


def _ipc_worker(rank, world, port, q):
    try:
        import torch
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        R, C = 3001, 70
        m = _matrix(R, C, 11)
        ev = Evaluator(0)
        b, e = row_range(R, rank, world)
        ev.upload(np.ascontiguousarray(m[b:e]), row_base=b)
        ev.prepare(0.03)
        h = ev.xchg_create(world, rank, 4096)
        handles = [None] * world
        dist.all_gather_object(handles, h)
        ev.xchg_open(handles)
        ok = True
        for step in range(3):
            pop = synth.random_population(3000, C, 2, 7, seed=100 + step)
            d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
            d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
            out = torch.empty(len(pop), dtype=torch.int32, device="cuda")
            dist.barrier()
            ev.evaluate_population_rows_sum_device(d_c.data_ptr(), d_o.data_ptr(), len(pop), out.data_ptr(),
                                                   TrendParams(0.03, step == 1))
            ev.sync()
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, 0.03, step == 1)
            ok &= bool(np.array_equal(out.cpu().numpy().view(np.uint32), want))
        dist.barrier()
        ev.close()
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(exc)))


def test_rows_sum_two_processes_ipc():
    import multiprocessing as mp

    build.build_ext()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in results), results


def _ranks(world, R, C, m, max_cand=5000):
    evs = [Evaluator(0) for _ in range(world)]
    for g, ev in enumerate(evs):
        b, e = row_range(R, g, world)
        ev.upload(np.ascontiguousarray(m[b:e]), row_base=b)
        ev.prepare(0.03)
        ev.xchg_create(world, g, max_cand)
    wins = [ev.xchg_window() for ev in evs]
    for ev in evs:
        ev.xchg_open_local(wins)
    return evs


@pytest.mark.parametrize("world", [2, 3])
def test_rows_sum_pipelined_steps(world):
    """Several steps issued back to back with no host sync: step k's exchange
    runs on the exchange stream while step k+1's count runs (two local ring
    slots, two inbox parities); every step's sums are exact."""
    import torch

    build.build_ext()
    R, C = 3333, 80
    m = _matrix(R, C, 40 + world)
    evs = _ranks(world, R, C, m)
    try:
        streams = [torch.cuda.Stream() for _ in range(world)]
        steps = []
        for step in range(7):
            pop = synth.random_population(3000 + 37 * step, C, 2, 7, seed=200 + step)
            approx, neg = ((0.03, False), (0.0, True), (0.1, False))[step % 3]
            d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
            d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
            outs = [torch.full((len(pop),), -1, dtype=torch.int32, device="cuda") for _ in range(world)]
            steps.append((pop, approx, neg, d_c, d_o, outs))
        torch.cuda.synchronize()
        for pop, approx, neg, d_c, d_o, outs in steps:
            for g, ev in enumerate(evs):
                ev.evaluate_population_rows_sum_async(d_c.data_ptr(), d_o.data_ptr(), len(pop), outs[g].data_ptr(),
                                                      TrendParams(approx, neg), stream=streams[g].cuda_stream)
        for g, ev in enumerate(evs):
            ev.xchg_fence(streams[g].cuda_stream)
        for ev in evs:
            ev.sync()
        for k, (pop, approx, neg, _, _, outs) in enumerate(steps):
            want = oracle.evaluate_population(m, pop.cols, pop.offsets, approx, neg)
            for g in range(world):
                np.testing.assert_array_equal(outs[g].cpu().numpy().view(np.uint32), want,
                                              err_msg=f"rank {g} step {k}")
    finally:
        for ev in evs:
            ev.close()


def test_window_header_mismatch_rejected():
    """Windows created with different max_cand (or world) cannot be mapped:
    a push would land outside the smaller peer's inbox."""
    build.build_ext()
    m = _matrix(600, 20, 1)
    evs = [Evaluator(0) for _ in range(2)]
    try:
        for g, ev in enumerate(evs):
            b, e = row_range(600, g, 2)
            ev.upload(np.ascontiguousarray(m[b:e]), row_base=b)
        evs[0].xchg_create(2, 0, 4096)
        evs[1].xchg_create(2, 1, 8192)
        wins = [ev.xchg_window() for ev in evs]
        for ev in evs:
            with pytest.raises(EbicError, match="max_cand"):
                ev.xchg_open_local(wins)
        evs[1].xchg_create(3, 1, 4096)
        with pytest.raises(EbicError, match="world"):
            evs[0].xchg_open_local([evs[0].xchg_window(), evs[1].xchg_window()])
    finally:
        for ev in evs:
            ev.close()


def test_failed_count_poisons_every_rank():
    """A rank whose count fails still runs the exchange (zeros + poison), so the
    epochs stay aligned; every rank's counts become the 0xFFFFFFFF sentinel
    and ebic_ctx_sync reports the failure on every rank."""
    import torch

    build.build_ext()
    R, C = 1200, 30
    m = _matrix(R, C, 5)
    evs = _ranks(2, R, C, m, max_cand=2000)
    try:
        pop = synth.random_population(1000, C, 2, 6, seed=1)
        d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
        d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
        outs = [torch.zeros(len(pop), dtype=torch.int32, device="cuda") for _ in range(2)]
        streams = [torch.cuda.Stream() for _ in range(2)]
        with pytest.raises(EbicError, match="approx"):  # rank 0: a count that cannot run
            evs[0].evaluate_population_rows_sum_async(d_c.data_ptr(), d_o.data_ptr(), len(pop), outs[0].data_ptr(),
                                                      TrendParams(float("nan")), stream=streams[0].cuda_stream)
        evs[1].evaluate_population_rows_sum_async(d_c.data_ptr(), d_o.data_ptr(), len(pop), outs[1].data_ptr(),
                                                  TrendParams(0.03), stream=streams[1].cuda_stream)
        for ev in evs:
            with pytest.raises(EbicError, match="poisoned"):
                ev.sync()
        for g in range(2):
            assert (outs[g].cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()
    finally:
        for ev in evs:
            ev.close()


def test_missing_peer_times_out_with_sentinel(monkeypatch):
    """A rank whose peer never arrives gives up after EBIC_XCHG_TIMEOUT_MS,
    writes the sentinel instead of stale counts and reports a timeout."""
    import torch

    monkeypatch.setenv("EBIC_XCHG_TIMEOUT_MS", "300")
    build.build_ext()
    R, C = 900, 25
    m = _matrix(R, C, 6)
    evs = _ranks(2, R, C, m, max_cand=1000)
    try:
        pop = synth.random_population(800, C, 2, 5, seed=2)
        d_c = torch.from_numpy(pop.cols.view(np.int32)).cuda()
        d_o = torch.from_numpy(pop.offsets.view(np.int32)).cuda()
        out = torch.full((len(pop),), 7, dtype=torch.int32, device="cuda")
        evs[0].evaluate_population_rows_sum_device(d_c.data_ptr(), d_o.data_ptr(), len(pop), out.data_ptr(),
                                                   TrendParams(0.03))
        with pytest.raises(EbicError, match="timed out"):
            evs[0].sync()
        assert (out.cpu().numpy().view(np.uint32) == 0xFFFFFFFF).all()
    finally:
        for ev in evs:
            ev.close()
