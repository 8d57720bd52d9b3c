"""CPU ORACLE for the fused-multiloop hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It loads ``oracle/build/liboracle.so``
(built from ``oracle/oracle.cpp`` by ``oracle/Makefile``); see ``oracle/oracle.h`` for the
reference file:line each function restates.  The product package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile liboracle.so (idempotent; make decides whether anything is stale)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        u64, i64, i32, c_int = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int
        L.orc_rng_advance.restype = u64
        L.orc_rng_advance.argtypes = [u64, u64]
        L.orc_rng_units.argtypes = [u64, u64, i64, _f64p, c_int]
        L.orc_rng_ints.argtypes = [u64, u64, i64, i64, _i64p, c_int]
        L.orc_kmeans_step.restype = c_int
        L.orc_kmeans_step.argtypes = [_f64p, i64, i32, i32, _f64p, _i64p, _i64p, _f64p, c_int, c_int]
        L.orc_kmeans_update.argtypes = [_i64p, _f64p, i32, i32, _f64p]
        L.orc_groupby_count.restype = c_int
        L.orc_groupby_count.argtypes = [_i64p, i64, i64, _i64p, c_int, c_int]
        L.orc_logreg_grad.restype = c_int
        L.orc_logreg_grad.argtypes = [_f64p, _i64p, i64, i32, _f64p, _f64p, c_int, c_int]
        L.orc_gda_pass1.restype = c_int
        L.orc_gda_pass1.argtypes = [_f64p, _i64p, i64, i32, _i64p, _f64p, _f64p, c_int, c_int]
        L.orc_gda_pass2.restype = c_int
        L.orc_gda_pass2.argtypes = [_f64p, _i64p, i64, i32, _f64p, _f64p, _f64p, c_int, c_int]
        L.orc_axpy.argtypes = [ctypes.c_double, _f64p, _f64p, i64, _f64p]
        L.orc_sum_f64.restype = ctypes.c_double
        L.orc_sum_f64.argtypes = [_f64p, i64, c_int, c_int]
        L.orc_sum_i64.restype = i64
        L.orc_sum_i64.argtypes = [_i64p, i64, c_int, c_int]
        L.orc_sum_sumsq_f64.argtypes = [_f64p, i64, _f64p, _f64p, c_int, c_int]
        L.orc_count_gt_f64.restype = i64
        L.orc_count_gt_f64.argtypes = [_f64p, i64, ctypes.c_double, c_int, c_int]
        L.orc_fnv64w.restype = u64
        L.orc_fnv64w.argtypes = [_i64p, i64]
        L.orc_format_double.restype = c_int
        L.orc_format_double.argtypes = [ctypes.c_double, ctypes.c_char_p]
        L.orc_num_threads.restype = c_int
        _lib = L
    return _lib


def _p(a: np.ndarray, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def threads() -> int:
    return int(lib().orc_num_threads())


# ---- Rng ---------------------------------------------------------------------------------

def rng_advance(state: int, n: int) -> int:
    return int(lib().orc_rng_advance(state, n))


def rng_units(seed: int, first_draw: int, n: int, nthreads: int | None = None) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().orc_rng_units(seed, first_draw, n, _p(out, _f64p), nthreads or threads())
    return out


def rng_ints(seed: int, first_draw: int, n: int, bound: int, nthreads: int | None = None) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    lib().orc_rng_ints(seed, first_draw, n, bound, _p(out, _i64p), nthreads or threads())
    return out


# ---- families ------------------------------------------------------------------------------

def kmeans_step(x: np.ndarray, k: int, mu: np.ndarray, workers: int = 1, chunks: int = 1):
    n, d = x.shape
    assign = np.empty(n, dtype=np.int64)
    counts = np.empty(k, dtype=np.int64)
    sums = np.empty((k, d), dtype=np.float64)
    rc = lib().orc_kmeans_step(_p(x, _f64p), n, d, k, _p(np.ascontiguousarray(mu), _f64p),
                               _p(assign, _i64p), _p(counts, _i64p), _p(sums, _f64p),
                               workers, chunks)
    assert rc == 0
    return assign, counts, sums


def kmeans_update(counts: np.ndarray, sums: np.ndarray) -> np.ndarray:
    k, d = sums.shape
    mu = np.empty((k, d), dtype=np.float64)
    with np.errstate(all="ignore"):
        lib().orc_kmeans_update(_p(counts, _i64p), _p(sums, _f64p), k, d, _p(mu, _f64p))
    return mu


def groupby_count(keys: np.ndarray, nbuckets: int, workers: int = 1, chunks: int = 1) -> np.ndarray:
    counts = np.empty(nbuckets, dtype=np.int64)
    rc = lib().orc_groupby_count(_p(keys, _i64p), keys.size, nbuckets, _p(counts, _i64p), workers, chunks)
    assert rc == 0
    return counts


def logreg_grad(x: np.ndarray, y: np.ndarray, theta: np.ndarray, workers: int = 1, chunks: int = 1):
    n, d = x.shape
    g = np.empty(d, dtype=np.float64)
    rc = lib().orc_logreg_grad(_p(x, _f64p), _p(y, _i64p), n, d, _p(np.ascontiguousarray(theta), _f64p),
                               _p(g, _f64p), workers, chunks)
    assert rc == 0
    return g


def gda_pass1(x: np.ndarray, y: np.ndarray, workers: int = 1, chunks: int = 1):
    n, d = x.shape
    n1 = np.zeros(1, dtype=np.int64)
    s0 = np.empty(d, dtype=np.float64)
    s1 = np.empty(d, dtype=np.float64)
    rc = lib().orc_gda_pass1(_p(x, _f64p), _p(y, _i64p), n, d, _p(n1, _i64p), _p(s0, _f64p),
                             _p(s1, _f64p), workers, chunks)
    assert rc == 0
    return int(n1[0]), s0, s1


def gda_pass2(x: np.ndarray, y: np.ndarray, mu0: np.ndarray, mu1: np.ndarray, workers: int = 1,
              chunks: int = 1) -> np.ndarray:
    n, d = x.shape
    s = np.empty((d, d), dtype=np.float64)
    rc = lib().orc_gda_pass2(_p(x, _f64p), _p(y, _i64p), n, d, _p(np.ascontiguousarray(mu0), _f64p),
                             _p(np.ascontiguousarray(mu1), _f64p), _p(s, _f64p), workers, chunks)
    assert rc == 0
    return s


def axpy(a: float, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    out = np.empty_like(x)
    lib().orc_axpy(a, _p(x, _f64p), _p(y, _f64p), x.size, _p(out, _f64p))
    return out


def sum_f64(x: np.ndarray, workers: int = 1, chunks: int = 1) -> float:
    return float(lib().orc_sum_f64(_p(x, _f64p), x.size, workers, chunks))


def sum_i64(x: np.ndarray, workers: int = 1, chunks: int = 1) -> int:
    return int(lib().orc_sum_i64(_p(x, _i64p), x.size, workers, chunks))


def sum_sumsq_f64(x: np.ndarray, workers: int = 1, chunks: int = 1):
    a = ctypes.c_double()
    b = ctypes.c_double()
    lib().orc_sum_sumsq_f64(_p(x, _f64p), x.size, ctypes.byref(a), ctypes.byref(b), workers, chunks)
    return a.value, b.value


def count_gt_f64(x: np.ndarray, thr: float, workers: int = 1, chunks: int = 1) -> int:
    return int(lib().orc_count_gt_f64(_p(x, _f64p), x.size, thr, workers, chunks))


# ---- utilities -----------------------------------------------------------------------------

def fnv64w(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.int64)
    return int(lib().orc_fnv64w(_p(v, _i64p), v.size))


def format_double(x: float) -> str:
    buf = ctypes.create_string_buffer(64)
    n = lib().orc_format_double(float(x), buf)
    return buf.raw[:n].decode()


def kmeans_canonical_text(counts: np.ndarray, mu: np.ndarray) -> str:
    """k count lines, then k*d format_double(mu[c][j]) lines (c-major)."""
    lines = [str(int(c)) for c in counts] + [format_double(v) for v in mu.reshape(-1)]
    return "".join(s + "\n" for s in lines)


def gda_canonical_text(n1: int, mu0: np.ndarray, mu1: np.ndarray, scatter: np.ndarray) -> str:
    """n1, then mu0[j], mu1[j] interleaved, then S row-major."""
    lines = [str(int(n1))]
    for j in range(mu0.size):
        lines.append(format_double(mu0[j]))
        lines.append(format_double(mu1[j]))
    lines += [format_double(v) for v in scatter.reshape(-1)]
    return "".join(s + "\n" for s in lines)


# ---- whole programs (the staged drivers of SURVEY App. A / B conventions) -------------------

def kmeans_inputs(n: int, d: int, k: int, seed: int = 1):
    """x = n*d next_unit() row-major (draws 0..n*d-1); mu0 = first k rows of x."""
    x = rng_units(seed, 0, n * d).reshape(n, d)
    return x, x[:k].copy()


def kmeans_run(x: np.ndarray, k: int, iters: int, mu0: np.ndarray, workers: int = 1, chunks: int = 1):
    """Free-running iterations; returns per-iteration (counts, fnv64w(assign), mu) history."""
    mu = mu0.copy()
    hist = []
    for _ in range(iters):
        assign, counts, sums = kmeans_step(x, k, mu, workers, chunks)
        mu = kmeans_update(counts, sums)
        hist.append((counts, fnv64w(assign), mu, sums, assign))
    return hist
