"""Break down the host-API (e2e) step time on the GPU box: where do the
microseconds between the kernel and the synchronous ebic_eval_counts go?"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2105_01196_b200 import Evaluator, TrendParams, synth  # noqa: E402

m, _ = synth.planted_trend_matrix(20000, 1000, 3, 500, 20, seed=1)
pops = [synth.random_population(16384, 1000, seed=42 + i) for i in range(4)]
ev = Evaluator(0)
ev.upload(m)
ev.prepare(0.03)
tp = TrendParams(0.03)
out = np.zeros(16384, dtype=np.uint32)


def timeit(label, fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{label:50s} {(time.perf_counter() - t0) / n * 1e3:8.3f} ms")


timeit("evaluate_population (host API, no flush)", lambda: ev.evaluate_population(pops[0], tp))
timeit("submit+wait raw", lambda: ev.wait(ev.submit(pops[0], out, tp)))
d_cols = torch.from_numpy(pops[0].cols.view(np.int32)).cuda()
d_offs = torch.from_numpy(pops[0].offsets.view(np.int32)).cuda()
d_cnt = torch.zeros(16384, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()


def dev():
    ev.evaluate_population_device(d_cols.data_ptr(), d_offs.data_ptr(), 16384, d_cnt.data_ptr(), tp,
                                  stream=s.cuda_stream)
    s.synchronize()


timeit("device API + stream sync", dev)


def dev_async():
    ev.evaluate_population_device(d_cols.data_ptr(), d_offs.data_ptr(), 16384, d_cnt.data_ptr(), tp,
                                  stream=s.cuda_stream)


timeit("device API launch only (async)", dev_async, n=200)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    for _ in range(3):
        dev_async()
    e0.record(s)
    for _ in range(20):
        dev_async()
    e1.record(s)
s.synchronize()
print(f"{'back-to-back kernel (events, L2 warm)':50s} {e0.elapsed_time(e1) / 20:8.3f} ms")
