"""Time the index build (rank plane + pair-trend index) at C3 / C2 shapes:
ebic_matrix_prepare with a fresh approx each time (forces a rebuild), wall
clock around a synchronised call, median of 7."""
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

from paper_2105_01196_b200 import Evaluator  # noqa: E402

for R, C in ((20000, 1000), (10000, 500), (100000, 2000)):
    ev = Evaluator(0)
    m = np.random.default_rng(1).standard_normal((R, C)).astype(np.float32)
    ev.upload(m)
    ts = []
    for k in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev.prepare(0.03 + 1e-4 * k)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{R} x {C}: prepare (plane + index) median {statistics.median(ts[1:]):.2f} ms  (all: {', '.join(f'{t:.2f}' for t in ts)})")
    ev.close()
