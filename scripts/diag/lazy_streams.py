"""Back-to-back device-API batches on the lazy index from several streams
(argv: R n_streams sync_every): which launches disagree with the oracle."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle  # noqa: E402
from paper_2105_01196_b200 import Evaluator, TrendParams, synth  # noqa: E402
from paper_2105_01196_b200._lib import EBIC_PATH_LAZY  # noqa: E402

R, n_streams, sync_every = (int(a) for a in sys.argv[1:4])
C = 400
rng = np.random.default_rng(11)
m = rng.standard_normal((R, C)).astype(np.float32)
m[: R // 3] = np.sort(m[: R // 3], axis=1)
m[rng.random(m.shape) < 0.03] = 0.0
ev = Evaluator(0)
ev.set_path(EBIC_PATH_LAZY)
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # earlier rounds: one stream, as a preceding test would
pops = [synth.random_population(5000, C, 2, 8, seed=300 + k) for k in range(6)]
want = [oracle.evaluate_population(m, p.cols, p.offsets, 0.03, True) for p in pops]
dev = [(torch.from_numpy(p.cols.view(np.int32)).cuda(), torch.from_numpy(p.offsets.view(np.int32)).cuda()) for p in pops]
outs = [torch.full((5000,), -1, dtype=torch.int32, device="cuda") for _ in range(18)]
for rnd in range(rounds - 1):
    ev.upload(m)
    s1 = torch.cuda.Stream()
    for i in range(18):
        dc, do = dev[i % 6]
        ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), 5000, outs[i].data_ptr(), TrendParams(0.03, True),
                                      stream=s1.cuda_stream)
    torch.cuda.synchronize()
    print("round", rnd, "(one stream) bad launches:",
          sum(int((outs[i].cpu().numpy().view(np.uint32) != want[i % 6]).any()) for i in range(18)), file=sys.stderr)
ev.upload(m)
streams = [torch.cuda.Stream() for _ in range(n_streams)]
torch.cuda.synchronize()
print("=== final round", file=sys.stderr)
for i in range(18):
    dc, do = dev[i % 6]
    ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), 5000, outs[i].data_ptr(), TrendParams(0.03, True),
                                  stream=streams[i % n_streams].cuda_stream)
    if sync_every and (i + 1) % sync_every == 0:
        torch.cuda.synchronize()
        print(i, ev.index_stats())
torch.cuda.synchronize()
ev.sync()
for i in range(18):
    got = outs[i].cpu().numpy().view(np.uint32)
    bad = np.nonzero(got != want[i % 6])[0]
    print("launch", i, "stream", i % n_streams, "bad", len(bad), "" if not len(bad) else
          f"first {bad[:5]} got {got[bad[:5]]} want {want[i % 6][bad[:5]]}")
print(ev.index_stats())
