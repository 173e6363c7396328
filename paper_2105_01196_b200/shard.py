"""Multi-GPU layer: one process per GPU (torch.distributed, NCCL over NVLink).

Two layouts; every (candidate, row) check is independent and
the only cross-unit combine is an integer sum per candidate, so both are exact
for any world size:

  rows  -- rank g holds matrix rows [g*R/G, (g+1)*R/G) as its own column-major
           store; every rank evaluates the WHOLE population on its shard and the
           partial uint32 counts are summed with one all_reduce(SUM) (the path's
           only real exchange).  Row lists (supporting_rows) are the per-shard
           ascending lists concatenated in rank order.
  pop   -- every rank holds the whole matrix (replicated); rank g evaluates
           its contiguous slice of the population; no reduction, counts are
           all-gathered only when every rank needs them.

Matrix source: every rank passes the host matrix (`source="local"`), or only
rank 0 does (`source="broadcast"`): the row-major matrix is then broadcast from
rank 0 -- over NVLink into each GPU's memory with NCCL, where each rank builds
its store straight from the device buffer (ebic_matrix_upload_device_*), or as
a CPU tensor with gloo.

Exchange of the rows layout: `exchange="collective"` sums the partial counts
with one all_reduce of the process group (NCCL over NVLink, or gloo);
`exchange="p2p"` sums them on the device through the exchange windows of
ebic_xchg.cuh (every rank's window mapped into every rank with CUDA IPC, one
fused push/wait/sum kernel, no collective call per step).

The evaluator itself is injected (`local`), so the sharding / exchange logic is
the same object in production (the CUDA `Evaluator`) and in the CPU gloo tests.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .trend import Population, TrendParams


def row_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row shard of rank `rank` (first n_rows % world ranks get one extra)."""
    base, extra = divmod(n_rows, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def pop_range(n_cand: int, rank: int, world: int) -> tuple[int, int]:
    return row_range(n_cand, rank, world)


def slice_population(pop: Population, begin: int, end: int) -> Population:
    o = pop.offsets
    cols = pop.cols[o[begin]:o[end]]
    offs = (o[begin:end + 1] - o[begin]).astype(np.uint32)
    return Population(cols, offs)


@dataclass
class ShardSpec:
    mode: str  # "rows" | "pop"
    rank: int
    world: int
    n_rows: int
    n_cols: int

    @property
    def rows(self) -> tuple[int, int]:
        return row_range(self.n_rows, self.rank, self.world) if self.mode == "rows" else (0, self.n_rows)


class ShardedEvaluator:
    """Host-facing sharded evaluation with the reference semantics of
    evaluate_population / supporting_rows (trend.cpp:48-72).

    `local` must provide upload(matrix, row_base=...), evaluate_population(pop, p)
    -> uint32 array and supporting_rows_batch(pop, p) -> list of arrays.
    `dist` is torch.distributed (already initialised) or None for world 1.
    """

    def __init__(self, local, matrix: np.ndarray | None, mode: str = "rows", dist=None, group=None,
                 source: str = "local", exchange: str = "collective", max_cand: int = 0):
        if mode not in ("rows", "pop"):
            raise ValueError("mode must be 'rows' or 'pop'")
        if source not in ("local", "broadcast"):
            raise ValueError("source must be 'local' or 'broadcast'")
        if exchange not in ("collective", "p2p"):
            raise ValueError("exchange must be 'collective' or 'p2p'")
        self.local = local
        self.dist = dist
        self.group = group
        self.exchange = exchange if mode == "rows" else "collective"
        world = dist.get_world_size(group) if dist is not None else 1
        rank = dist.get_rank(group) if dist is not None else 0
        if source == "broadcast" and world > 1:
            self._upload_broadcast(matrix, mode, rank, world)
        else:
            if matrix is None:
                raise ValueError("matrix is required with source='local'")
            self.spec = ShardSpec(mode, rank, world, int(matrix.shape[0]), int(matrix.shape[1]))
            b, e = self.spec.rows
            local.upload(np.ascontiguousarray(matrix[b:e]), row_base=b)
        if self.exchange == "p2p":
            if max_cand <= 0:
                raise ValueError("exchange='p2p' needs max_cand (the largest population per call)")
            self._setup_p2p(int(max_cand))

    @classmethod
    def attach(cls, local, n_rows: int, n_cols: int, mode: str = "rows", dist=None, group=None,
               exchange: str = "collective", max_cand: int = 0) -> "ShardedEvaluator":
        """Wrap a context that already holds this rank's shard (uploaded with
        row_base = row_range(...)[0]) and, for exchange='p2p', an opened
        exchange window of at least max_cand candidates."""
        self = cls.__new__(cls)
        self.local, self.dist, self.group = local, dist, group
        world = dist.get_world_size(group) if dist is not None else 1
        rank = dist.get_rank(group) if dist is not None else 0
        self.spec = ShardSpec(mode, rank, world, int(n_rows), int(n_cols))
        self.exchange = exchange if mode == "rows" else "collective"
        if self.exchange == "p2p":
            self._setup_p2p(int(max_cand), window_open=True)
        return self

    def _setup_p2p(self, max_cand: int, window_open: bool = False) -> None:
        """Create this rank's exchange window and map every peer's (IPC handles
        all-gathered once through the process group)."""
        import torch

        if not window_open:
            handle = self.local.xchg_create(self.spec.world, self.spec.rank, max_cand)
            handles = [handle]
            if self.dist is not None and self.spec.world > 1:
                handles = [None] * self.spec.world
                self.dist.all_gather_object(handles, handle, group=self.group)
            self.local.xchg_open(handles)
        self.max_cand = max_cand
        dev = torch.device("cuda", torch.cuda.current_device())
        self._dev = dev
        self._stream = torch.cuda.Stream(dev)
        self._h_counts = torch.empty(max_cand, dtype=torch.int32, pin_memory=True)
        self._d_counts = torch.empty(max_cand, dtype=torch.int32, device=dev)
        self._pinned = {}

    def _pin(self, key: str, a: np.ndarray):
        """Page-locked staging copy of a host array (grown on demand)."""
        import torch

        buf = self._pinned.get(key)
        if buf is None or buf.numel() < a.size:
            buf = torch.empty(max(a.size, 1024), dtype=torch.int32, pin_memory=True)
            self._pinned[key] = buf
        buf.numpy().view(np.uint32)[:a.size] = a
        return buf[:a.size]

    def _rows_sum_p2p(self, pop: Population, p: TrendParams) -> np.ndarray:
        import torch

        n = len(pop)
        if n > self.max_cand:
            raise ValueError(f"{n} candidates exceed the exchange window ({self.max_cand})")
        with torch.cuda.stream(self._stream):
            d_cols = self._pin("cols", pop.cols).to(self._dev, non_blocking=True)
            d_offs = self._pin("offs", pop.offsets).to(self._dev, non_blocking=True)
            self.local.evaluate_population_rows_sum_device(d_cols.data_ptr(), d_offs.data_ptr(), n,
                                                           self._d_counts.data_ptr(), p,
                                                           stream=self._stream.cuda_stream)
            self._h_counts[:n].copy_(self._d_counts[:n], non_blocking=True)
        self._stream.synchronize()
        self.local.sync()  # raises on a device-side error (bad column, exchange timeout / poison)
        return self._h_counts[:n].numpy().view(np.uint32).copy()

    def _upload_broadcast(self, matrix, mode, rank, world):
        """Rank 0's matrix to every rank (shape and dtype first), then each rank
        uploads its row block of the broadcast buffer."""
        import torch

        dist, group = self.dist, self.group
        dev = _collective_device(dist, group)
        src = dist.get_global_rank(group, 0) if group is not None else 0
        meta = torch.zeros(3, dtype=torch.int64)
        if rank == 0:
            if matrix is None:
                raise ValueError("rank 0 needs the matrix with source='broadcast'")
            m = np.asarray(matrix)
            meta = torch.tensor([m.shape[0], m.shape[1], int(m.dtype != np.float32)], dtype=torch.int64)
        meta = meta.to(dev)
        dist.broadcast(meta, src=src, group=group)
        n_rows, n_cols, f64 = (int(x) for x in meta.tolist())
        dtype = torch.float64 if f64 else torch.float32
        if rank == 0:
            buf = torch.from_numpy(np.ascontiguousarray(matrix, dtype=np.float64 if f64 else np.float32)).to(dev)
        else:
            buf = torch.empty((n_rows, n_cols), dtype=dtype, device=dev)
        dist.broadcast(buf, src=src, group=group)
        self.spec = ShardSpec(mode, rank, world, n_rows, n_cols)
        b, e = self.spec.rows
        block = buf[b:e]  # contiguous rows of a row-major buffer
        if block.is_cuda and hasattr(self.local, "upload_device"):
            torch.cuda.current_stream().synchronize()  # the broadcast has landed before the context's stream reads it
            self.local.upload_device(block.data_ptr(), e - b, n_cols, dtype="f64" if f64 else "f32", row_base=b)
        else:
            self.local.upload(block.cpu().numpy(), row_base=b)
        del buf, block

    # -- collectives (torch tensors on CPU for gloo, on CUDA for nccl) -------
    def _all_reduce_sum(self, counts: np.ndarray) -> np.ndarray:
        if self.dist is None or self.spec.world == 1:
            return counts
        import torch

        t = torch.from_numpy(counts.astype(np.int64))
        dev = _collective_device(self.dist, self.group)
        t = t.to(dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy().astype(np.uint32)

    def _all_gather_var(self, arr: np.ndarray) -> list[np.ndarray]:
        if self.dist is None or self.spec.world == 1:
            return [arr]
        objs = [None] * self.spec.world
        self.dist.all_gather_object(objs, arr, group=self.group)
        return objs

    # -- reference API ---------------------------------------------------------
    def evaluate_population(self, pop: Population, p: TrendParams | None = None) -> np.ndarray:
        p = p or TrendParams()
        if self.spec.mode == "rows":
            if self.exchange == "p2p":
                return self._rows_sum_p2p(pop, p)
            return self._all_reduce_sum(self.local.evaluate_population(pop, p))
        b, e = pop_range(len(pop), self.spec.rank, self.spec.world)
        mine = self.local.evaluate_population(slice_population(pop, b, e), p)
        return np.concatenate(self._all_gather_var(mine)).astype(np.uint32)

    def supporting_rows_batch(self, pop: Population, p: TrendParams | None = None) -> list[np.ndarray]:
        p = p or TrendParams()
        if self.spec.mode == "pop":
            # every rank holds the whole matrix: rank 0's answer is the answer
            return self.local.supporting_rows_batch(pop, p)
        mine = self.local.supporting_rows_batch(pop, p)  # global row ids, ascending per shard
        parts = self._all_gather_var(mine)
        # shards are contiguous and in rank order, so concatenation stays ascending
        return [np.concatenate([parts[r][i] for r in range(self.spec.world)]).astype(np.uint32)
                for i in range(len(pop))]


def _collective_device(dist, group):
    backend = dist.get_backend(group)
    if backend == "nccl":
        import torch

        return torch.device("cuda", torch.cuda.current_device())
    return "cpu"
