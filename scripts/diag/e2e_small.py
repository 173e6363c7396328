"""Host-API latency of one evaluate_population call at small batch sizes
(pinned [offsets | cols] block, counts into pinned memory), with the inputs
DMA'd (EBIC_ZC_READ_MAX=0) or read in place by the kernel.  Prints the
median / p10 of 300 calls per config and the cost of a no-op ctypes call."""
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2105_01196_b200 import Evaluator, Population, TrendParams  # noqa: E402


def pinned(a):
    t = torch.empty(a.size, dtype=torch.int32, pin_memory=True)
    v = t.numpy().view(np.uint32)
    v[:] = a
    return t, v


for name in sys.argv[1:] or ["spec", "c2", "c3"]:
    cfg = bench.CONFIGS[name]
    m, pops = bench.make_inputs(cfg, 2)
    ev = Evaluator(0)
    ev.upload(m)
    ev.prepare(cfg["approx"])
    tp = TrendParams(cfg["approx"], cfg["negative"])
    p = pops[0]
    keep, blk = pinned(np.concatenate([p.offsets, p.cols]))
    n1 = p.offsets.size
    pp = Population(blk[n1:], blk[:n1])
    keep2, out = pinned(np.zeros(len(p), dtype=np.uint32))
    for _ in range(50):
        ev.evaluate_population(pp, tp, out=out)
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        ev.evaluate_population(pp, tp, out=out)
        ts.append((time.perf_counter() - t0) * 1e6)
    nop = []
    for _ in range(300):
        t0 = time.perf_counter()
        ev.launch_count()
        nop.append((time.perf_counter() - t0) * 1e6)
    ts.sort()
    print(f"{name} P={len(p)} in_bytes={4 * blk.size} zc_read_max={os.environ.get('EBIC_ZC_READ_MAX', '0')}: "
          f"median {statistics.median(ts):.1f} us, p10 {ts[30]:.1f} us; no-op ctypes call {statistics.median(nop):.1f} us")
    ev.close()
