"""Cold start on the device clock: fresh context per repetition (argv[1] config, argv[2] reps), the first
evaluate_population_device batch timed with CUDA events (after a warm-up context so clocks are up)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
from paper_2105_01196_b200 import Evaluator, TrendParams  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m, pops = bench.make_inputs(cfg, 2)
tp = TrendParams(cfg["approx"], cfg["negative"])
d = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda(), len(p))
     for p in pops]
out = torch.zeros(cfg["pop"], dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()  # (not the legacy default stream: the library would take its own stream for 0)
x = torch.randn(8192, 8192, device="cuda")
for r in range(reps + 1):
    ev = Evaluator(0)
    ev.upload(m)
    ev.set_lazy_build(int(sys.argv[3]) if len(sys.argv) > 3 else 0)
    for _ in range(20):
        x = x @ x.T * 1e-4  # keep clocks up
    torch.cuda.synchronize()
    ts = []
    for k in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dc, do, n = d[min(k, 1)]
        e0.record(s)
        ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, out.data_ptr(), tp, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    if r:
        print("first %.3f ms, new population %.3f ms, repeat %.3f ms" % tuple(ts), ev.index_stats()["lazy_slots_used"])
    del ev
