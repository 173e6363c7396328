"""Cold start at C3 (or argv[1]): fresh context, upload, first / second evaluate_population through the
host API -- run under `ncu --metrics gpu__time_duration.sum` to see which kernels make up the first call."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2105_01196_b200 import Evaluator, TrendParams  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
m, pops = bench.make_inputs(cfg, 2)
tp = TrendParams(cfg["approx"], cfg["negative"])
torch.zeros(1, device="cuda")
ev = Evaluator(0)
ev.upload(m)
torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter()
    got = ev.evaluate_population(pops[i % 2], tp)
    print("call", i, "%.3f ms" % ((time.perf_counter() - t0) * 1e3), ev.index_stats())
