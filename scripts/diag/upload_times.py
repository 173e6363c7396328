"""Host -> device matrix upload times (fresh context each, then a second
upload on the same context): f32 and f64, 20k x 1000 and 200k x 2000."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2105_01196_b200 import Evaluator  # noqa: E402

for R, C in ((20_000, 1000), (200_000, 2000)):
    for dt in (np.float32, np.float64):
        m = np.random.default_rng(1).standard_normal((R, C)).astype(dt)
        ev = Evaluator(0)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ev.upload(m)
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{R} x {C} {np.dtype(dt).name} ({m.nbytes / 1e9:.2f} GB): upload ms first {ts[0]:.1f}, then {ts[1]:.1f}, {ts[2]:.1f}")
        ev.close()
