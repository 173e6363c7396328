"""One rank's share of a row-sharded step (C3 by default; argv[1] = config), measured on one GPU: the count
kernel over R/N rows (N = 1, 2, 4, 8) for the whole 16384-candidate
population, back-to-back device-API batches (the same stream mode as the
bench) -- the per-rank compute floor a row-sharded step cannot go below."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2105_01196_b200 import Evaluator, TrendParams  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
m, pops = bench.make_inputs(cfg, 4)
tp = TrendParams(cfg["approx"], cfg["negative"])
for n in (1, 2, 4, 8):
    rows = cfg["rows"] // n
    ev = Evaluator(0)
    ev.upload(np.ascontiguousarray(m[:rows]))
    ev.prepare(cfg["approx"])
    d = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda()) for p in pops]
    out = torch.zeros(cfg["pop"], dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    for i in range(8):
        ev.evaluate_population_device(d[i % 4][0].data_ptr(), d[i % 4][1].data_ptr(), cfg["pop"], out.data_ptr(), tp,
                                      stream=s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 200
    e0.record(s)
    for i in range(steps):
        ev.evaluate_population_device(d[i % 4][0].data_ptr(), d[i % 4][1].data_ptr(), cfg["pop"], out.data_ptr(), tp,
                                      stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ev.sync()
    us = e0.elapsed_time(e1) * 1e3 / steps
    print(f"N={n}: {rows} rows per rank, {us:.1f} us per back-to-back step "
          f"({cfg['pop'] / us * 1e6:.3g} evals/s per rank; index {ev.index_info()[0] / 1e6:.0f} MB)")
    ev.close()
