"""Parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg (and its
`--impl reference` arm) may import this package.  The product
(paper_2105_01196_b200) never does.

  port()       ctypes binding of oracle/liboracle.so, the C restatement of
               trend.cpp (trend_oracle.c).  Built on demand with gcc.
  reference()  ctypes binding of oracle/_ref/libbicseek_ref.so: the UNMODIFIED
               reference sources + ref_capi.cpp glue (built only where
               /root/reference exists; the built file travels to the GPU box).
"""
from __future__ import annotations

import ctypes as C
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libbicseek_ref.so"
_lock = threading.Lock()
_port = None
_ref = None

_vp = C.c_void_p


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def port():
    """The C restatement (builds liboracle.so with gcc if missing or stale)."""
    global _port
    with _lock:
        if _port is None:
            src = HERE / "trend_oracle.c"
            if not PORT_SO.exists() or PORT_SO.stat().st_mtime < src.stat().st_mtime:
                subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
            L = C.CDLL(str(PORT_SO))
            L.oracle_row_supports.restype = C.c_int
            L.oracle_row_supports.argtypes = [_vp, C.c_uint64, C.c_uint64, _vp, C.c_uint32, C.c_double, C.c_int]
            L.oracle_supporting_rows.restype = C.c_uint64
            L.oracle_supporting_rows.argtypes = [_vp, C.c_uint64, C.c_uint64, _vp, C.c_uint32, C.c_double,
                                                 C.c_int, _vp, C.c_uint64]
            L.oracle_evaluate_population.restype = None
            L.oracle_evaluate_population.argtypes = [_vp, C.c_uint64, C.c_uint64, _vp, _vp, C.c_uint64,
                                                     C.c_double, C.c_int, _vp, C.c_int]
            L.oracle_evaluate_population_f32.restype = None
            L.oracle_evaluate_population_f32.argtypes = L.oracle_evaluate_population.argtypes
            L.oracle_fitness.restype = C.c_double
            L.oracle_fitness.argtypes = [C.c_uint64] * 4
            L.oracle_threads.restype = C.c_int
            _port = L
    return _port


def reference_available() -> bool:
    return REF_SO.exists()


def reference():
    """The unmodified reference library (raises if oracle/_ref was not built)."""
    global _ref
    with _lock:
        if _ref is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
            L = C.CDLL(str(REF_SO))
            L.ref_last_error.restype = C.c_char_p
            L.ref_gen_background.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _vp]
            L.ref_gen_scenario.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                           C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_int, _vp]
            L.ref_init_population.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp]
            L.ref_matrix_create.restype = _vp
            L.ref_matrix_create.argtypes = [_vp, C.c_uint64, C.c_uint64]
            L.ref_matrix_destroy.argtypes = [_vp]
            L.ref_population_create.restype = _vp
            L.ref_population_create.argtypes = [_vp, _vp, C.c_uint64]
            L.ref_population_destroy.argtypes = [_vp]
            L.ref_pool_create.restype = _vp
            L.ref_pool_create.argtypes = [C.c_uint]
            L.ref_pool_destroy.argtypes = [_vp]
            L.ref_pool_size.restype = C.c_uint
            L.ref_pool_size.argtypes = [_vp]
            L.ref_evaluate_population.argtypes = [_vp, _vp, C.c_double, C.c_int, _vp, _vp]
            L.ref_supporting_rows.restype = C.c_int64
            L.ref_supporting_rows.argtypes = [_vp, _vp, C.c_uint32, C.c_double, C.c_int, _vp, C.c_uint64]
            L.ref_row_supports.argtypes = [_vp, C.c_uint64, _vp, C.c_uint32, C.c_double, C.c_int]
            L.ref_fitness.restype = C.c_double
            L.ref_fitness.argtypes = [C.c_uint64] * 4
            L.ref_test_chromosomes.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp]
            if hasattr(L, "ref_parse_matrix_tsv"):  # io.cpp compiled in (needs nlohmann json.hpp at build)
                L.ref_parse_matrix_tsv.argtypes = [C.c_char_p, _vp, C.c_uint64, C.POINTER(C.c_uint64),
                                                   C.POINTER(C.c_uint64)]
                L.ref_write_matrix_tsv.argtypes = [C.c_char_p, _vp, C.c_uint64, C.c_uint64]
            _ref = L
    return _ref


# ---------------------------------------------------------------------------
# numpy-level helpers over the C restatement ("port")
# ---------------------------------------------------------------------------
def _csr(cols, offsets):
    return np.ascontiguousarray(cols, dtype=np.uint32), np.ascontiguousarray(offsets, dtype=np.uint32)


def evaluate_population(m: np.ndarray, cols, offsets, approx: float, negative: bool, threads: int = 0) -> np.ndarray:
    """trend.cpp:56-72 restated in C.  m: (R, C) float64 or float32, row-major."""
    L = port()
    cols, offsets = _csr(cols, offsets)
    n = offsets.size - 1
    out = np.zeros(n, dtype=np.uint32)
    if m.dtype == np.float32:
        m = np.ascontiguousarray(m)
        L.oracle_evaluate_population_f32(_p(m), m.shape[0], m.shape[1], _p(cols), _p(offsets), n, approx,
                                         int(negative), _p(out), int(threads))
    else:
        m = np.ascontiguousarray(m, dtype=np.float64)
        L.oracle_evaluate_population(_p(m), m.shape[0], m.shape[1], _p(cols), _p(offsets), n, approx,
                                     int(negative), _p(out), int(threads))
    return out


def supporting_rows(m: np.ndarray, seq, approx: float, negative: bool) -> np.ndarray:
    L = port()
    m = np.ascontiguousarray(m, dtype=np.float64)
    seq = np.ascontiguousarray(seq, dtype=np.uint32)
    out = np.empty(m.shape[0], dtype=np.uint32)
    n = L.oracle_supporting_rows(_p(m), m.shape[0], m.shape[1], _p(seq), seq.size, approx, int(negative),
                                 _p(out), out.size)
    return out[:n].copy()


def row_supports(m: np.ndarray, row: int, seq, approx: float, negative: bool) -> bool:
    L = port()
    m = np.ascontiguousarray(m, dtype=np.float64)
    seq = np.ascontiguousarray(seq, dtype=np.uint32)
    return bool(L.oracle_row_supports(_p(m), m.shape[1], int(row), _p(seq), seq.size, approx, int(negative)))


def fitness(count: int, ncols: int, min_rows: int = 10, col_cap: int = 8) -> float:
    return float(port().oracle_fitness(count, ncols, min_rows, col_cap))


# ---------------------------------------------------------------------------
# helpers over the unmodified reference
# ---------------------------------------------------------------------------
class RefMatrix:
    """An ExpressionMatrix owned by the reference library."""

    def __init__(self, m: np.ndarray):
        self.L = reference()
        self.values = np.ascontiguousarray(m, dtype=np.float64)
        self.h = self.L.ref_matrix_create(_p(self.values), self.values.shape[0], self.values.shape[1])
        if not self.h:
            raise ValueError(self.L.ref_last_error().decode())

    def __del__(self):
        try:
            self.L.ref_matrix_destroy(self.h)
        except Exception:
            pass


class RefPopulation:
    def __init__(self, cols, offsets):
        self.L = reference()
        self.cols, self.offsets = _csr(cols, offsets)
        self.n = self.offsets.size - 1
        self.h = self.L.ref_population_create(_p(self.cols), _p(self.offsets), self.n)

    def __del__(self):
        try:
            self.L.ref_population_destroy(self.h)
        except Exception:
            pass


class RefPool:
    def __init__(self, threads: int = 0):
        self.L = reference()
        self.h = self.L.ref_pool_create(int(threads))
        self.size = int(self.L.ref_pool_size(self.h))

    def __del__(self):
        try:
            self.L.ref_pool_destroy(self.h)
        except Exception:
            pass


def ref_evaluate(mat: RefMatrix, pop: RefPopulation, approx: float, negative: bool, pool: RefPool | None = None):
    out = np.zeros(pop.n, dtype=np.uint32)
    st = mat.L.ref_evaluate_population(mat.h, pop.h, approx, int(negative), pool.h if pool else None, _p(out))
    if st:
        raise RuntimeError(mat.L.ref_last_error().decode())
    return out


def ref_supporting_rows(mat: RefMatrix, seq, approx: float, negative: bool) -> np.ndarray:
    seq = np.ascontiguousarray(seq, dtype=np.uint32)
    out = np.empty(mat.values.shape[0], dtype=np.uint32)
    n = mat.L.ref_supporting_rows(mat.h, _p(seq), seq.size, approx, int(negative), _p(out), out.size)
    if n < 0:
        raise RuntimeError(mat.L.ref_last_error().decode())
    return out[:n].copy()


def ref_gen_background(rows: int, cols: int, seed: int, quantize: bool = False) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    L = reference()
    if L.ref_gen_background(rows, cols, seed, int(quantize), _p(out)):
        raise RuntimeError(L.ref_last_error().decode())
    return out


SCENARIOS = ["six_types", "overlap", "narrow", "noise", "colincrease", "colin1000", "different", "large_variant"]
PATTERNS = ["trend", "column_const", "row_const", "shift", "scale", "shift_scale"]


def ref_gen_scenario(rows, cols, bic_rows, bic_cols, num_bics, seed, scenario="six_types", pattern="trend",
                     noise=0.0, mean_shift=0.0, quantize=True) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    L = reference()
    if L.ref_gen_scenario(SCENARIOS.index(scenario), PATTERNS.index(pattern), rows, cols, bic_rows, bic_cols,
                          num_bics, noise, mean_shift, seed, int(quantize), _p(out)):
        raise RuntimeError(L.ref_last_error().decode())
    return out


def ref_init_population(pop_size: int, num_cols: int, seed: int = 42, len_min: int = 3, len_max: int = 5):
    L = reference()
    cols = np.empty(pop_size * len_max, dtype=np.uint32)
    offs = np.empty(pop_size + 1, dtype=np.uint32)
    if L.ref_init_population(pop_size, num_cols, seed, len_min, len_max, _p(cols), _p(offs)):
        raise RuntimeError(L.ref_last_error().decode())
    return cols[:offs[-1]].copy(), offs


def ref_test_chromosomes(seed: int, n: int, num_cols: int):
    L = reference()
    cols = np.empty(n * 7, dtype=np.uint32)
    offs = np.empty(n + 1, dtype=np.uint32)
    L.ref_test_chromosomes(seed, n, num_cols, _p(cols), _p(offs))
    return cols[:offs[-1]].copy(), offs


class RefParseError(Exception):
    """The reference parser's ParseError (message verbatim)."""


def ref_io_available() -> bool:
    return reference_available() and hasattr(reference(), "ref_parse_matrix_tsv")


def ref_parse_matrix_tsv(path) -> np.ndarray:
    """The reference TSV reader (io.cpp:78-111): row-major float64 values."""
    L = reference()
    r, c = C.c_uint64(0), C.c_uint64(0)
    st = L.ref_parse_matrix_tsv(str(path).encode(), None, 0, C.byref(r), C.byref(c))
    if st == 1:
        raise RefParseError(L.ref_last_error().decode())
    out = np.empty((r.value, c.value), dtype=np.float64)
    if L.ref_parse_matrix_tsv(str(path).encode(), _p(out), out.size, C.byref(r), C.byref(c)):
        raise RefParseError(L.ref_last_error().decode())
    return out


def ref_write_matrix_tsv(path, m: np.ndarray) -> None:
    """The reference TSV writer (io.cpp:113-130, %.17g, labels r0../c0..)."""
    L = reference()
    m = np.ascontiguousarray(m, dtype=np.float64)
    if L.ref_write_matrix_tsv(str(path).encode(), _p(m), m.shape[0], m.shape[1]):
        raise RuntimeError(L.ref_last_error().decode())

