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
                 source: str = "local"):
        if mode not in ("rows", "pop"):
            raise ValueError("mode must be 'rows' or 'pop'")
        if source not in ("local", "broadcast"):
            raise ValueError("source must be 'local' or 'broadcast'")
        self.local = local
        self.dist = dist
        self.group = group
        world = dist.get_world_size(group) if dist is not None else 1
        rank = dist.get_rank(group) if dist is not None else 0
        if source == "broadcast" and world > 1:
            self._upload_broadcast(matrix, mode, rank, world)
            return
        if matrix is None:
            raise ValueError("matrix is required with source='local'")
        self.spec = ShardSpec(mode, rank, world, int(matrix.shape[0]), int(matrix.shape[1]))
        b, e = self.spec.rows
        local.upload(np.ascontiguousarray(matrix[b:e]), row_base=b)

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
