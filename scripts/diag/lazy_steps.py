"""Per-step timing of back-to-back device-API batches on the lazy index
(diagnostic for the bench's stream mode): events around every step, host
time per call, index stats before / after."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2105_01196_b200 import Evaluator, TrendParams  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
use_torch_stream = "--ctx-stream" not in sys.argv
m, pops = bench.make_inputs(cfg, 4)
ev = Evaluator(0)
ev.upload(m)
ev.prepare(cfg["approx"])
tp = TrendParams(cfg["approx"], cfg["negative"])
d = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda(), len(p))
     for p in pops]
out = torch.zeros(cfg["pop"], dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
sp = s.cuda_stream if use_torch_stream else None
for phase in ("warm", "timed", "timed2"):
    n = 8 if phase == "warm" else int(sys.argv[2]) if len(sys.argv) > 2 else 20
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    host = []
    torch.cuda.synchronize()
    for i in range(n):
        dc, do, k = d[i % 4]
        evs[i][0].record(s)
        t0 = time.perf_counter()
        ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), k, out.data_ptr(), tp, stream=sp)
        host.append((time.perf_counter() - t0) * 1e3)
        evs[i][1].record(s)
    torch.cuda.synchronize()
    ev.sync()
    print(phase, "device ms:", " ".join("%.2f" % a.elapsed_time(b) for a, b in evs))
    print(phase, "host ms:  ", " ".join("%.2f" % h for h in host))
    print(phase, ev.index_stats())
