"""Matrix ingest on the GPU box's host: the reference parse_matrix_tsv
(io.cpp:78-111, one thread) vs ebic_tsv_read (all host threads) on a TSV
written by the reference writer, and the full load into the device store
(parse into page-locked memory + upload + f32-exactness check + transpose)."""
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_2105_01196_b200 import Evaluator, read_matrix_tsv, synth  # noqa: E402


def timed(fn, reps=3):
    best = 1e9
    out = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        best = min(best, time.perf_counter() - t0)
    return best, out


for rows, cols in ((20000, 1000), (10000, 500)):
    m = synth.planted_trend_matrix(rows, cols, 3, 500, 20, seed=1)[0].astype(np.float64)
    with tempfile.TemporaryDirectory() as d:
        f = Path(d) / "m.tsv"
        oracle.ref_write_matrix_tsv(f, m)
        mb = f.stat().st_size / 1e6
        t_ref, ref = timed(lambda: oracle.ref_parse_matrix_tsv(f), reps=2)
        t_1, one = timed(lambda: read_matrix_tsv(f, threads=1))
        t_all, got = timed(lambda: read_matrix_tsv(f, threads=0))
        same = np.array_equal(got.view(np.uint64), ref.view(np.uint64)) and np.array_equal(one, ref)
        ev = Evaluator(0)
        t_load, _ = timed(lambda: ev.load_tsv(f))
        ev.close()
        print(f"{rows} x {cols} ({mb:.0f} MB TSV, {os.cpu_count()} host threads): reference parse {t_ref:.3f} s | "
              f"ebic_tsv_read 1 thread {t_1:.3f} s, all threads {t_all:.3f} s ({t_ref / t_all:.1f}x) | "
              f"load into the device store {t_load:.3f} s | values bit-identical: {same}", flush=True)
