"""Where do the microseconds of one host-API step (ebic_eval_counts with
pinned host arrays) go on the GPU box?  C3 shapes (20k x 1000, P = 16384)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2105_01196_b200 import Evaluator, Population, TrendParams, synth  # noqa: E402

m, _ = synth.planted_trend_matrix(20000, 1000, 3, 500, 20, seed=1)
pop = synth.random_population(16384, 1000, seed=42)
ev = Evaluator(0)
ev.upload(m)
ev.prepare(0.03)
tp = TrendParams(0.03)


def pinned(a):
    t = torch.empty(a.size, dtype=torch.int32, pin_memory=True)
    v = t.numpy().view(np.uint32)
    v[:] = a
    return t, v


tc, vc = pinned(pop.cols)
to, vo = pinned(pop.offsets)
tout, vout = pinned(np.zeros(16384, np.uint32))
ppop = Population(vc, vo)
tiny = Population(np.array([0, 1, 2], np.uint32), np.array([0, 3], np.uint32))


def timeit(label, fn, n=100):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{label:60s} {(time.perf_counter() - t0) / n * 1e6:9.1f} us", flush=True)


tb, vb = pinned(np.concatenate([pop.offsets, pop.cols]))
bpop = Population(vb[pop.offsets.size:], vb[: pop.offsets.size])
timeit("host API, pinned [offsets|cols] block (bench e2e)", lambda: ev.evaluate_population(bpop, tp, out=vout))
timeit("host API, pinned separate arrays", lambda: ev.evaluate_population(ppop, tp, out=vout))
timeit("host API, pageable arrays (marshaller)", lambda: ev.evaluate_population(pop, tp))
timeit("host API, 1 candidate x 3 cols (fixed overhead)", lambda: ev.evaluate_population(tiny, tp))
d_c = torch.empty(vc.size, dtype=torch.int32, device="cuda")
d_o = torch.empty(vo.size, dtype=torch.int32, device="cuda")
d_n = torch.zeros(16384, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s):
        d_c.copy_(tc, non_blocking=True)
        d_o.copy_(to, non_blocking=True)
    s.synchronize()


def d2h():
    with torch.cuda.stream(s):
        tout.copy_(d_n, non_blocking=True)
    s.synchronize()


timeit("torch H2D cols+offsets (327 KB) + sync", h2d)
timeit("torch D2H counts (64 KB) + sync", d2h)
timeit("empty stream sync", lambda: s.synchronize())
h2d()


def dev():
    ev.evaluate_population_device(d_c.data_ptr(), d_o.data_ptr(), 16384, d_n.data_ptr(), tp, stream=s.cuda_stream)
    s.synchronize()


timeit("device API + sync (kernel + launch)", dev)

# the same zero-copy call straight through ctypes (no Python-side checks)
import ctypes as C  # noqa: E402

L, h = ev._L, ev._h
pc, po, pout = C.c_void_p(bpop.cols.ctypes.data), C.c_void_p(bpop.offsets.ctypes.data), C.c_void_p(vout.ctypes.data)
timeit("raw ctypes ebic_eval_counts, pinned block", lambda: L.ebic_eval_counts(h, pc, po, 16384, 0.03, 0, pout))
timeit("raw ctypes, 1 candidate (fixed overhead)",
       lambda: L.ebic_eval_counts(h, C.c_void_p(tiny.cols.ctypes.data), C.c_void_p(tiny.offsets.ctypes.data), 1,
                                  0.03, 0, pout))
# host-side validation cost: offsets scan only (ebic_eval_counts with an invalid approx fails after nothing)
t0 = time.perf_counter()
for _ in range(1000):
    np.all(np.diff(bpop.offsets.astype(np.int64)) > 0)
print(f"{'numpy offsets scan (reference point)':60s} {(time.perf_counter() - t0) / 1000 * 1e6:9.1f} us")
