"""Python mirror of the reference trend/fitness API (proj/include/bicseek/trend.hpp)
over the B200 evaluator.

Reference interface -> this module
  TrendParams            trend.hpp:13-25 (validate trend.cpp:8-13)  -> TrendParams
  row_supports           trend.hpp:30-31 / trend.cpp:41-46           -> row_supports / Evaluator.row_supports
  supporting_rows        trend.hpp:33-35 / trend.cpp:48-54           -> supporting_rows / Evaluator.supporting_rows
  evaluate_population    trend.hpp:37-45 / trend.cpp:56-72           -> evaluate_population / Evaluator.evaluate_population
  fitness                trend.hpp:47-50 / trend.cpp:74-79           -> fitness
  ExpressionMatrix       matrix.hpp:13-43 (row-major double)         -> numpy (R, C) array, uploaded once per Evaluator
  Chromosome             bicluster.hpp:13-24                         -> sequence of ints / Population (CSR)

Same names, argument meaning and error behaviour (ValueError for what the
reference raises std::invalid_argument for).  Every evaluating call runs on the
GPU through libebic.so; there is no CPU path in this module.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import EBIC_STORE_AUTO, EBIC_STORE_F32, EBIC_STORE_F64, EbicError, check


@dataclass
class TrendParams:
    """trend.hpp:13-25."""

    approx: float = 0.03
    negative_trends: bool = False
    min_rows: int = 10
    col_cap: int = 8

    def validate(self) -> None:  # trend.cpp:8-13
        if not (self.approx >= 0.0 and self.approx < 1.0):
            raise ValueError("TrendParams: approx must be in [0, 1)")
        if self.min_rows < 2:
            raise ValueError("TrendParams: min_rows must be >= 2")
        if self.col_cap < 2:
            raise ValueError("TrendParams: col_cap must be >= 2")


_DEFAULT_PARAMS = TrendParams()


class Population:
    """A batch of candidate column sequences in CSR form (uint32 cols, uint32 offsets)."""

    __slots__ = ("cols", "offsets")

    def __init__(self, cols: np.ndarray, offsets: np.ndarray):
        self.cols = np.ascontiguousarray(cols, dtype=np.uint32)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
        if self.offsets.ndim != 1 or self.offsets.size < 1 or self.offsets[0] != 0:
            raise ValueError("Population: offsets must start at 0")
        if int(self.offsets[-1]) != self.cols.size:
            raise ValueError("Population: offsets[-1] must equal len(cols)")

    @classmethod
    def from_sequences(cls, seqs: Iterable[Sequence[int]]) -> "Population":
        seqs = [list(s) for s in seqs]
        offs = np.zeros(len(seqs) + 1, dtype=np.uint32)
        if seqs:
            offs[1:] = np.cumsum([len(s) for s in seqs])
        cols = np.fromiter((c for s in seqs for c in s), dtype=np.int64, count=int(offs[-1]))
        if cols.size and (cols.min() < 0 or cols.max() >= 2**32):
            raise ValueError("Population: column index out of range")
        return cls(cols.astype(np.uint32), offs)

    def __len__(self) -> int:
        return self.offsets.size - 1

    def sequence(self, i: int) -> np.ndarray:
        return self.cols[self.offsets[i]:self.offsets[i + 1]]

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)


def _as_population(pop) -> Population:
    if isinstance(pop, Population):
        return pop
    return Population.from_sequences(pop)


def _ptr(a: np.ndarray) -> int:
    # the buffer address as a plain int (the bindings declare c_void_p); cheaper
    # than ndarray.ctypes.data_as on the per-call path
    return a.__array_interface__["data"][0]


def device_count() -> int:
    n = C.c_int(0)
    check(_lib.lib().ebic_device_count(C.byref(n)))
    return n.value


class Evaluator:
    """One device context + one resident matrix (or row shard).

    The matrix is stored column-major in HBM: float32 when every value is
    float32-representable (always for float32 input), otherwise float64, so
    results are bit-exact with the reference for any finite input.
    """

    def __init__(self, device: int = 0):
        self._L = _lib.lib()
        h = C.c_void_p()
        check(self._L.ebic_ctx_create(int(device), C.byref(h)))
        self._h = h
        self.device = device
        self.n_rows = 0
        self.n_cols = 0
        self.row_base = 0
        self.store = 0

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.ebic_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_stream(self, cuda_stream: int | None) -> None:
        check(self._L.ebic_ctx_set_stream(self._h, C.c_void_p(cuda_stream or 0)))

    def sync(self) -> None:
        check(self._L.ebic_ctx_sync(self._h))

    def launch_count(self) -> int:
        n = C.c_uint64(0)
        check(self._L.ebic_ctx_launch_count(self._h, C.byref(n)))
        return n.value

    def set_slab_rows(self, slab_rows: int) -> None:
        check(self._L.ebic_ctx_set_slab_rows(self._h, int(slab_rows)))

    def set_path(self, path: int) -> None:
        """EBIC_PATH_AUTO (rank-plane slab kernel when C <= 8192) / _VALUE / _PLANE."""
        check(self._L.ebic_ctx_set_path(self._h, int(path)))

    def set_pair_layout(self, pairs_per_lane: int = 0, cands_per_warp: int = 0) -> None:
        """Force one packed-pair layout of the hot kernel ((0, 0) = auto)."""
        check(self._L.ebic_ctx_set_pair_layout(self._h, int(pairs_per_lane), int(cands_per_warp)))

    def set_table_budget(self, nbytes: int) -> None:
        """Memory cap of the pair-trend index (AUTO path uses it only below the cap)."""
        check(self._L.ebic_ctx_set_table_budget(self._h, int(nbytes)))

    def set_lazy_build(self, mode: int = 0) -> None:
        """Lazy index build route: 0 auto (cold batches build first), 1 inside the count kernel, 2 build pass first."""
        check(self._L.ebic_ctx_set_lazy_build(self._h, int(mode)))

    def index_info(self) -> tuple[int, bool]:
        """(bytes the pair-trend index of the resident matrix needs, whether it is built)."""
        nb, used = C.c_uint64(0), C.c_int(0)
        check(self._L.ebic_matrix_index_info(self._h, C.byref(nb), C.byref(used)))
        return int(nb.value), bool(used.value)

    # -- row-shard exchange over peer memory (ebic.h, ebic_xchg.cuh) ------------
    def xchg_create(self, world: int, rank: int, max_cand: int) -> bytes:
        """Allocate this rank's exchange window; returns its CUDA IPC handle."""
        h = C.create_string_buffer(64)
        check(self._L.ebic_xchg_create(self._h, int(world), int(rank), int(max_cand), h))
        return h.raw

    def xchg_open(self, handles: Sequence[bytes]) -> None:
        """Map the peers' windows from their IPC handles (rank order)."""
        buf = C.create_string_buffer(b"".join(bytes(h).ljust(64, b"\0")[:64] for h in handles), 64 * len(handles))
        check(self._L.ebic_xchg_open(self._h, buf))

    def xchg_open_local(self, windows: Sequence[int]) -> None:
        """Map windows of contexts in this process (device pointers, rank order)."""
        arr = (C.c_void_p * len(windows))(*[int(w) for w in windows])
        check(self._L.ebic_xchg_open_local(self._h, arr))

    def xchg_window(self) -> int:
        p = C.c_void_p(0)
        check(self._L.ebic_xchg_window(self._h, C.byref(p)))
        return int(p.value or 0)

    def xchg_destroy(self) -> None:
        check(self._L.ebic_xchg_destroy(self._h))

    def evaluate_population_rows_sum_device(self, d_cols: int, d_offsets: int, n_cand: int, d_counts: int,
                                            params: TrendParams | None = None, stream: int | None = None) -> None:
        """Row-sharded step: this shard's counts summed over all ranks through peer memory."""
        p = params or TrendParams()
        check(self._L.ebic_eval_counts_rows_sum(self._h, C.c_void_p(d_cols), C.c_void_p(d_offsets), int(n_cand),
                                                float(p.approx), int(bool(p.negative_trends)),
                                                C.c_void_p(d_counts), C.c_void_p(stream or 0)))

    def evaluate_population_rows_sum_async(self, d_cols: int, d_offsets: int, n_cand: int, d_counts: int,
                                           params: TrendParams | None = None, stream: int | None = None) -> None:
        """Pipelined row-sharded step: the count runs on `stream`, the exchange on the
        context's exchange stream; d_counts is complete after xchg_fence(stream) / sync()."""
        p = params or TrendParams()
        check(self._L.ebic_eval_counts_rows_sum_async(self._h, C.c_void_p(d_cols), C.c_void_p(d_offsets),
                                                      int(n_cand), float(p.approx), int(bool(p.negative_trends)),
                                                      C.c_void_p(d_counts), C.c_void_p(stream or 0)))

    def xchg_fence(self, stream: int | None = None) -> None:
        """Order `stream` after every exchange issued so far."""
        check(self._L.ebic_xchg_fence(self._h, C.c_void_p(stream or 0)))

    def load_tsv(self, path, threads: int = 0, store: int = EBIC_STORE_AUTO) -> tuple[int, int, int]:
        """Parse a reference-format TSV matrix (io.cpp:78-111) on all host threads
        straight into page-locked memory and upload it; returns (rows, cols, store)."""
        st, r, c = C.c_int(0), C.c_uint64(0), C.c_uint64(0)
        check(self._L.ebic_matrix_load_tsv(self._h, str(path).encode(), int(threads), int(store), C.byref(st),
                                           C.byref(r), C.byref(c)))
        self.n_rows, self.n_cols = int(r.value), int(c.value)
        return int(r.value), int(c.value), int(st.value)

    def prepare(self, approx: float) -> None:
        """Build the rank plane for `approx` now (otherwise built on first use)."""
        check(self._L.ebic_matrix_prepare(self._h, float(approx)))

    def index_stats(self) -> dict:
        """The index behind the last evaluation: mode ('none' | 'full' | 'lazy'), full-index
        bytes, lazy pool fill / capacity / bytes, vectors built lazily, pool resets."""
        mode = C.c_int(0)
        v = [C.c_uint64(0) for _ in range(6)]
        check(self._L.ebic_matrix_index_stats(self._h, C.byref(mode), *[C.byref(x) for x in v]))
        return {"mode": ("none", "full", "lazy")[mode.value], "full_bytes": v[0].value,
                "lazy_slots_used": v[1].value, "lazy_slots_cap": v[2].value, "lazy_bytes": v[3].value,
                "lazy_built": v[4].value, "lazy_resets": v[5].value}

    def build_info(self) -> dict:
        """One-time costs (ms) of the last preparation: index allocation, rank plane, pair-trend index."""
        a, pl, ix = C.c_double(0), C.c_double(0), C.c_double(0)
        check(self._L.ebic_matrix_build_info(self._h, C.byref(a), C.byref(pl), C.byref(ix)))
        return {"alloc_ms": a.value, "plane_ms": pl.value, "index_ms": ix.value}

    # -- matrix store ------------------------------------------------------
    def upload(self, matrix: np.ndarray, row_base: int = 0, store: int = EBIC_STORE_AUTO) -> int:
        """Upload a row-major (R, C) matrix (float64 or float32).  Returns the store mode."""
        m = np.asarray(matrix)
        if m.ndim != 2:
            raise ValueError("matrix must be 2-D (rows, cols)")
        if m.dtype == np.float32:
            m = np.ascontiguousarray(m)
            if store == EBIC_STORE_F64:
                m = m.astype(np.float64)
            else:
                check(self._L.ebic_matrix_upload_f32(self._h, _ptr(m), m.shape[0], m.shape[1], row_base))
                self._set_shape(m.shape, row_base, EBIC_STORE_F32)
                return EBIC_STORE_F32
        m = np.ascontiguousarray(m, dtype=np.float64)
        out = C.c_int(0)
        check(self._L.ebic_matrix_upload_f64(self._h, _ptr(m), m.shape[0], m.shape[1], row_base,
                                             int(store), C.byref(out)))
        self._set_shape(m.shape, row_base, out.value)
        return out.value

    def upload_device(self, ptr: int, n_rows: int, n_cols: int, dtype: str = "f32", row_base: int = 0,
                      store: int = EBIC_STORE_AUTO) -> int:
        """Upload a row-major matrix already in this context's GPU memory (device
        pointer `ptr`, e.g. a torch CUDA tensor an NCCL broadcast filled)."""
        if dtype == "f32":
            check(self._L.ebic_matrix_upload_device_f32(self._h, int(ptr), int(n_rows), int(n_cols), int(row_base)))
            self._set_shape((n_rows, n_cols), row_base, EBIC_STORE_F32)
            return EBIC_STORE_F32
        if dtype != "f64":
            raise ValueError("dtype must be 'f32' or 'f64'")
        out = C.c_int(0)
        check(self._L.ebic_matrix_upload_device_f64(self._h, int(ptr), int(n_rows), int(n_cols), int(row_base),
                                                    int(store), C.byref(out)))
        self._set_shape((n_rows, n_cols), row_base, out.value)
        return out.value

    def _set_shape(self, shape, row_base, store):
        self.n_rows, self.n_cols = int(shape[0]), int(shape[1])
        self.row_base = int(row_base)
        self.store = int(store)

    def matrix_info(self) -> dict:
        r, c, ld, rb = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        st = C.c_int()
        check(self._L.ebic_matrix_info(self._h, C.byref(r), C.byref(c), C.byref(ld), C.byref(st), C.byref(rb)))
        return {"rows": r.value, "cols": c.value, "ld": ld.value, "store": st.value, "row_base": rb.value}

    # -- evaluation --------------------------------------------------------
    def evaluate_population(self, pop, params: TrendParams | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """trend.cpp:56-72: uint32 support count per candidate (host arrays, synchronous).

        If the population arrays and `out` are page-locked (e.g. numpy views of
        torch pin_memory tensors), the library DMAs them directly (no staging copy).
        """
        p = params or _DEFAULT_PARAMS
        if type(pop) is not Population:
            pop = _as_population(pop)
        n = pop.offsets.size - 1
        if out is None:
            out = np.zeros(n, dtype=np.uint32)
        elif out.dtype != np.uint32 or not out.flags.c_contiguous or out.size < n:
            raise ValueError("out must be a contiguous uint32 array of at least len(pop) elements")
        if n == 0:
            return out
        check(self._L.ebic_eval_counts(self._h, _ptr(pop.cols), _ptr(pop.offsets), n,
                                       float(p.approx), int(bool(p.negative_trends)), _ptr(out)))
        return out

    def evaluate_population_device(self, d_cols: int, d_offsets: int, n_cand: int, d_counts: int,
                                   params: TrendParams | None = None, stream: int | None = None) -> None:
        """Device pointers (e.g. torch tensors' data_ptr()), asynchronous on `stream`."""
        p = params or TrendParams()
        check(self._L.ebic_eval_counts_device(self._h, C.c_void_p(d_cols), C.c_void_p(d_offsets), int(n_cand),
                                              float(p.approx), int(bool(p.negative_trends)),
                                              C.c_void_p(d_counts), C.c_void_p(stream or 0)))

    def submit(self, pop: Population, out: np.ndarray, params: TrendParams | None = None) -> int:
        """Batch marshaller: async evaluation; `out` (uint32, len(pop)) is filled by wait()."""
        p = params or TrendParams()
        if out.dtype != np.uint32 or out.size < len(pop) or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous uint32 array of len(pop)")
        t = C.c_uint64(0)
        check(self._L.ebic_eval_submit(self._h, _ptr(pop.cols), _ptr(pop.offsets), len(pop), float(p.approx),
                                       int(bool(p.negative_trends)), _ptr(out), C.byref(t)))
        return t.value

    def wait(self, ticket: int) -> None:
        check(self._L.ebic_eval_wait(self._h, int(ticket)))

    def supporting_rows(self, chromosome: Sequence[int], params: TrendParams | None = None) -> np.ndarray:
        """trend.cpp:48-54: ascending (global) rows supporting one candidate."""
        p = params or TrendParams()
        cols = np.ascontiguousarray(chromosome, dtype=np.uint32)
        rows = np.empty(max(self.n_rows, 1), dtype=np.uint32)
        n = C.c_uint64(0)
        check(self._L.ebic_support_rows(self._h, _ptr(cols), cols.size, float(p.approx),
                                        int(bool(p.negative_trends)), _ptr(rows), rows.size, C.byref(n)))
        return rows[:n.value].copy()

    def supporting_rows_batch(self, pop, params: TrendParams | None = None) -> list[np.ndarray]:
        p = params or TrendParams()
        pop = _as_population(pop)
        n = len(pop)
        offs = np.zeros(n + 1, dtype=np.uint64)
        cap = 0
        rows = np.empty(1, dtype=np.uint32)
        while True:
            st = self._L.ebic_support_rows_batch(self._h, _ptr(pop.cols), _ptr(pop.offsets), n, float(p.approx),
                                                 int(bool(p.negative_trends)), _ptr(rows), cap, _ptr(offs))
            if st == _lib.EBIC_ERR_CAPACITY:
                cap = int(offs[-1])
                rows = np.empty(max(cap, 1), dtype=np.uint32)
                continue
            check(st)
            break
        return [rows[offs[i]:offs[i + 1]].copy() for i in range(n)]

    def support_overlaps(self, pop, params: TrendParams | None = None) -> tuple[np.ndarray, np.ndarray]:
        """Row-set sizes and pairwise intersections of a batch without row lists
        (the |rows_a n rows_b| of induced_jaccard, evolution.cpp:44-51):
        returns (sizes[n], inter[n, n]) as uint64."""
        p = params or TrendParams()
        pop = _as_population(pop)
        n = len(pop)
        sizes = np.zeros(n, dtype=np.uint64)
        inter = np.zeros((n, n), dtype=np.uint64)
        check(self._L.ebic_support_overlap_batch(self._h, _ptr(pop.cols), _ptr(pop.offsets), n, float(p.approx),
                                                  int(bool(p.negative_trends)), _ptr(sizes), _ptr(inter)))
        return sizes, inter

    def row_supports(self, row: int, chromosome: Sequence[int], params: TrendParams | None = None) -> bool:
        p = params or TrendParams()
        cols = np.ascontiguousarray(chromosome, dtype=np.uint32)
        out = C.c_int(0)
        check(self._L.ebic_row_supports(self._h, int(row), _ptr(cols), cols.size, float(p.approx),
                                        int(bool(p.negative_trends)), C.byref(out)))
        return bool(out.value)


# ---------------------------------------------------------------------------
# free functions with the reference signatures (matrix passed on every call;
# a module-level Evaluator caches the device copy, keyed by identity AND
# content, exactly like the C++ drop-in TU)
# ---------------------------------------------------------------------------
_default: Evaluator | None = None
_default_key = None


def _bind(m: np.ndarray) -> Evaluator:
    global _default, _default_key
    m = np.asarray(m)
    if _default is None:
        _default = Evaluator(0)
    key = (m.dtype.str, m.shape)
    if _default_key is None or _default_key[0] != key or not np.array_equal(_default_key[1], m):
        _default.upload(m)
        _default_key = (key, m.copy())
    return _default


def row_supports(m: np.ndarray, row: int, c: Sequence[int], p: TrendParams) -> bool:
    return _bind(m).row_supports(row, c, p)


def supporting_rows(m: np.ndarray, c: Sequence[int], p: TrendParams) -> np.ndarray:
    return _bind(m).supporting_rows(c, p)


def evaluate_population(m: np.ndarray, pop, p: TrendParams, pool=None) -> np.ndarray:
    """`pool` (the reference WorkerPool) is accepted and ignored: the GPU grid replaces it."""
    return _bind(m).evaluate_population(pop, p)


def fitness(support_count: int, num_cols: int, p: TrendParams) -> float:
    """trend.cpp:74-79 (exact: count * 2^min(num_cols, col_cap), 0 below min_rows)."""
    return float(_lib.lib().ebic_fitness(int(support_count), int(num_cols), int(p.min_rows), int(p.col_cap)))


__all__ = [
    "TrendParams", "Population", "Evaluator", "EbicError", "device_count",
    "row_supports", "supporting_rows", "evaluate_population", "fitness",
    "EBIC_STORE_AUTO", "EBIC_STORE_F32", "EBIC_STORE_F64",
]


def read_matrix_tsv(path, threads: int = 0) -> np.ndarray:
    """The reference's TSV matrix format (io.cpp:78-111) parsed on all host
    threads (no device needed); same values and error messages."""
    L = _lib.lib()
    r, c = C.c_uint64(0), C.c_uint64(0)
    st = L.ebic_tsv_read(str(path).encode(), int(threads), None, 0, C.byref(r), C.byref(c))
    if st != _lib.EBIC_ERR_CAPACITY:
        check(st)
    out = np.empty((r.value, c.value), dtype=np.float64)
    check(L.ebic_tsv_read(str(path).encode(), int(threads), _ptr(out) if out.size else None, out.size,
                          C.byref(r), C.byref(c)))
    return out

