"""Host-side mirror of the fused-multiloop families, over the dlx C ABI.

Device memory and streams are torch CUDA tensors / streams (plumbing only); every kernel is
one of libdlx.so's hand-written sm_100a kernels, called through ``include/dlx.h``.  The
function names follow the reference's vector DSL and loop constructors:

==========================  ===============================================================
this module                 reference (/root/reference/proj)
==========================  ===============================================================
``rng_units/rng_ints``      ``vec_rand`` / ``vec_rand_int`` + ``Rng`` (vectordsl.cpp:10-20,
                            runtime.hpp:86-96)
``map_axpy``                ``DVec::zip_with`` collect (vectordsl.cpp:113-119)
``reduce_sum``              ``DVec::sum`` reduce (vectordsl.cpp:121-131)
``mean_variance``           ``mean`` + ``variance`` fused into one loop (vectordsl.cpp:167-184)
``count_where_gt``          ``DVec::count_where`` predicated reduce (vectordsl.cpp:138-151)
``kmeans_step``             one fused k-means multiloop
``groupby_count``           K predicated count reduces
``logreg_grad``             fused dot -> sigmoid -> d reduces
``gda``                     GDA passes 1 and 2
==========================  ===============================================================
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import check

_F64 = torch.float64
_I64 = torch.int64


def _dev(device=None) -> torch.device:
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Workspace:
    """Caller-owned scratch for the launchers (they never allocate)."""

    def __init__(self):
        self._bufs: dict[torch.device, torch.Tensor] = {}

    def get(self, nbytes: int, device) -> tuple[ctypes.c_void_p, int]:
        device = _dev(device)
        buf = self._bufs.get(device)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
            self._bufs[device] = buf
        return ctypes.c_void_p(buf.data_ptr()), buf.numel()


_WS = Workspace()


# ---- synthetic sources -------------------------------------------------------------------

def rng_units(n: int, seed: int = 1, first_draw: int = 0, device=None, out=None) -> torch.Tensor:
    L = _lib.load()
    out = out if out is not None else torch.empty(n, dtype=_F64, device=_dev(device))
    check(L.dlx_rng_units(_ptr(out), n, seed, first_draw, _stream()))
    return out


def rng_ints(n: int, bound: int, seed: int = 1, first_draw: int = 0, device=None, out=None) -> torch.Tensor:
    L = _lib.load()
    out = out if out is not None else torch.empty(n, dtype=_I64, device=_dev(device))
    check(L.dlx_rng_ints(_ptr(out), n, bound, seed, first_draw, _stream()))
    return out


# ---- generic collect / reduce ----------------------------------------------------------------

def map_axpy(a: float, x: torch.Tensor, y: torch.Tensor, out=None) -> torch.Tensor:
    L = _lib.load()
    out = out if out is not None else torch.empty_like(x)
    check(L.dlx_map_axpy(float(a), _ptr(x), _ptr(y), x.numel(), _ptr(out), _stream()))
    return out


def _reduce(fn: str, x: torch.Tensor, out: torch.Tensor, *extra):
    L = _lib.load()
    ws, wsb = _WS.get(L.dlx_reduce_workspace_bytes(x.numel()), x.device)
    args = [_ptr(x), x.numel(), *extra, _ptr(out), ws, wsb, _stream()]
    check(getattr(L, fn)(*args))
    return out


def reduce_sum(x: torch.Tensor) -> torch.Tensor:
    if x.dtype == _I64:
        return _reduce("dlx_reduce_sum_i64", x, torch.empty(1, dtype=_I64, device=x.device))
    return _reduce("dlx_reduce_sum_f64", x, torch.empty(1, dtype=_F64, device=x.device))


def mean_variance(x: torch.Tensor) -> tuple[float, float]:
    """One fused loop with two reduce elems (sum, sum of squares); the reference's
    ``variance`` is E[x^2] - mean^2 (vectordsl.cpp:176-184)."""
    s = _reduce("dlx_reduce_sum_sumsq_f64", x, torch.empty(2, dtype=_F64, device=x.device)).cpu()
    n = float(x.numel())
    mean = float(s[0]) / n
    return mean, float(s[1]) / n - mean * mean


def count_where_gt(x: torch.Tensor, thr: float) -> torch.Tensor:
    L = _lib.load()
    out = torch.empty(1, dtype=_I64, device=x.device)
    ws, wsb = _WS.get(L.dlx_reduce_workspace_bytes(x.numel()), x.device)
    check(L.dlx_reduce_count_gt_f64(_ptr(x), x.numel(), float(thr), _ptr(out), ws, wsb, _stream()))
    return out


# ---- k-means -----------------------------------------------------------------------------------

def kmeans_step(x: torch.Tensor, mu: torch.Tensor, assign: torch.Tensor | None = None,
                counts: torch.Tensor | None = None, sums: torch.Tensor | None = None,
                method: int = _lib.KMEANS_AUTO, want_assign: bool = True):
    """One fused k-means multiloop on the local shard: (assign int32 | None, counts, sums)."""
    L = _lib.load()
    n, d = x.shape
    k = mu.shape[0]
    dev = x.device
    if want_assign and assign is None:
        assign = torch.empty(n, dtype=torch.int32, device=dev)
    counts = counts if counts is not None else torch.empty(k, dtype=_I64, device=dev)
    sums = sums if sums is not None else torch.empty((k, d), dtype=_F64, device=dev)
    ws, wsb = _WS.get(L.dlx_kmeans_workspace_bytes(n, d, k), dev)
    check(L.dlx_kmeans_step(_ptr(x), n, d, k, _ptr(mu), _ptr(assign) if want_assign else None,
                            _ptr(counts), _ptr(sums), ws, wsb, method, _stream()))
    return (assign if want_assign else None), counts, sums


def kmeans_iteration(x: torch.Tensor, mu: torch.Tensor, assign: torch.Tensor | None = None,
                     counts: torch.Tensor | None = None, sums: torch.Tensor | None = None,
                     method: int = _lib.KMEANS_AUTO, want_assign: bool = True):
    """kmeans_step + kmeans_update in place on mu, the update fused into the combine launch
    (dlx_kmeans_iteration): (assign int32 | None, counts, sums); mu holds the new centroids."""
    L = _lib.load()
    n, d = x.shape
    k = mu.shape[0]
    dev = x.device
    if want_assign and assign is None:
        assign = torch.empty(n, dtype=torch.int32, device=dev)
    counts = counts if counts is not None else torch.empty(k, dtype=_I64, device=dev)
    sums = sums if sums is not None else torch.empty((k, d), dtype=_F64, device=dev)
    ws, wsb = _WS.get(L.dlx_kmeans_workspace_bytes(n, d, k), dev)
    check(L.dlx_kmeans_iteration(_ptr(x), n, d, k, _ptr(mu), _ptr(assign) if want_assign else None,
                                 _ptr(counts), _ptr(sums), ws, wsb, method, _stream()))
    return (assign if want_assign else None), counts, sums


def kmeans_update(counts: torch.Tensor, sums: torch.Tensor, mu: torch.Tensor | None = None) -> torch.Tensor:
    L = _lib.load()
    k, d = sums.shape
    mu = mu if mu is not None else torch.empty_like(sums)
    check(L.dlx_kmeans_update(_ptr(counts), _ptr(sums), k, d, _ptr(mu), _stream()))
    return mu


def kmeans_last_recheck_count(n: int, d: int, k: int, device=None) -> int:
    """Samples the last screened step (shape n, d, k) re-evaluated with the exact chain."""
    L = _lib.load()
    ws, _ = _WS.get(L.dlx_kmeans_workspace_bytes(n, d, k), _dev(device))
    v = ctypes.c_int64()
    check(L.dlx_kmeans_last_recheck_count(ws, n, d, k, ctypes.byref(v), _stream()))
    return v.value


# ---- GroupBy -------------------------------------------------------------------------------------

def groupby_count(keys: torch.Tensor, nbuckets: int, out: torch.Tensor | None = None) -> torch.Tensor:
    L = _lib.load()
    out = out if out is not None else torch.empty(nbuckets, dtype=_I64, device=keys.device)
    ws, wsb = _WS.get(L.dlx_groupby_workspace_bytes(keys.numel(), nbuckets), keys.device)
    check(L.dlx_groupby_count(_ptr(keys), keys.numel(), nbuckets, _ptr(out), ws, wsb, _stream()))
    return out


# ---- logistic regression ---------------------------------------------------------------------------

def logreg_grad(x: torch.Tensor, y: torch.Tensor, theta: torch.Tensor, out=None) -> torch.Tensor:
    L = _lib.load()
    n, d = x.shape
    out = out if out is not None else torch.empty(d, dtype=_F64, device=x.device)
    ws, wsb = _WS.get(L.dlx_logreg_workspace_bytes(n, d), x.device)
    # float32 x: the fp32-storage opt-in (exact promotion, fp64 arithmetic, rows.cu)
    fn = L.dlx_logreg_grad_f32 if x.dtype == torch.float32 else L.dlx_logreg_grad
    check(fn(_ptr(x), _ptr(y), n, d, _ptr(theta), _ptr(out), ws, wsb, _stream()))
    return out


def axpy_inplace(theta: torch.Tensor, grad: torch.Tensor, alpha: float) -> torch.Tensor:
    L = _lib.load()
    check(L.dlx_axpy_inplace(_ptr(theta), _ptr(grad), float(alpha), theta.numel(), _stream()))
    return theta


# ---- GDA ---------------------------------------------------------------------------------------------

def gda_pass1(x: torch.Tensor, y: torch.Tensor):
    L = _lib.load()
    n, d = x.shape
    n1 = torch.empty(1, dtype=_I64, device=x.device)
    s0 = torch.empty(d, dtype=_F64, device=x.device)
    s1 = torch.empty(d, dtype=_F64, device=x.device)
    ws, wsb = _WS.get(L.dlx_gda_workspace_bytes(n, d), x.device)
    check(L.dlx_gda_pass1(_ptr(x), _ptr(y), n, d, _ptr(n1), _ptr(s0), _ptr(s1), ws, wsb, _stream()))
    return n1, s0, s1


def gda_means(n1, s0, s1, n_total: int):
    L = _lib.load()
    d = s0.numel()
    mu0 = torch.empty_like(s0)
    mu1 = torch.empty_like(s1)
    check(L.dlx_gda_means(_ptr(n1), _ptr(s0), _ptr(s1), n_total, d, _ptr(mu0), _ptr(mu1), _stream()))
    return mu0, mu1


def gda_pass2(x: torch.Tensor, y: torch.Tensor, mu0: torch.Tensor, mu1: torch.Tensor, out=None):
    L = _lib.load()
    n, d = x.shape
    out = out if out is not None else torch.empty((d, d), dtype=_F64, device=x.device)
    ws, wsb = _WS.get(L.dlx_gda_workspace_bytes(n, d), x.device)
    check(L.dlx_gda_pass2(_ptr(x), _ptr(y), n, d, _ptr(mu0), _ptr(mu1), _ptr(out), ws, wsb, _stream()))
    return out


def gda_fit(x: torch.Tensor, y: torch.Tensor):
    """Single-pass fit (d <= 64, csrc/gda_dmma.cu): n1, mu0, mu1, S from one read of x."""
    L = _lib.load()
    n, d = x.shape
    n1 = torch.empty(1, dtype=_I64, device=x.device)
    mu0 = torch.empty(d, dtype=_F64, device=x.device)
    mu1 = torch.empty(d, dtype=_F64, device=x.device)
    S = torch.empty((d, d), dtype=_F64, device=x.device)
    ws, wsb = _WS.get(L.dlx_gda_fit_workspace_bytes(n, d), x.device)
    check(L.dlx_gda_fit(_ptr(x), _ptr(y), n, d, _ptr(n1), _ptr(mu0), _ptr(mu1), _ptr(S), ws, wsb, _stream()))
    return n1, mu0, mu1, S


def gda_fit_last_fallback(x: torch.Tensor) -> bool:
    """Whether the last gda_fit on x's shape took the exact-means fallback (synchronises)."""
    L = _lib.load()
    n, d = x.shape
    ws, _ = _WS.get(L.dlx_gda_fit_workspace_bytes(n, d), x.device)
    flag = ctypes.c_int(0)
    check(L.dlx_gda_fit_last_fallback(ws, n, d, ctypes.byref(flag)))
    return bool(flag.value)


def gda_fit_path(x: torch.Tensor, y: torch.Tensor) -> str:
    """The first pass dlx_gda_fit runs for (x, y): "int8" (tcgen05 kind::i8), "dmma" (k-split
    fp64 tensor cores) or "rowblocks"."""
    L = _lib.load()
    n, d = x.shape
    path = ctypes.c_int(0)
    check(L.dlx_gda_fit_path(_ptr(x), _ptr(y), n, d, ctypes.byref(path)))
    return {2: "int8", 1: "dmma", 0: "rowblocks"}[path.value]


def gda(x: torch.Tensor, y: torch.Tensor, comm=None):
    """phi-numerator n1, mu0, mu1 and the unnormalised scatter S.  One
    device-local fit reads x once (gda_fit); sharded fits run the two reference passes with
    the class sums and the scatter summed across ranks in between."""
    n_local, d = x.shape
    if d <= 64:
        n1, mu0, mu1, S = gda_fit(x, y)
        if comm is None:
            return n1, mu0, mu1, S
        # sharded: pool the ranks' fits (csrc/gda_dmma.cu, gda_combine_ranks_kernel)
        L = _lib.load()
        w = 2 + 2 * d
        table = torch.zeros((comm.world, w), dtype=_F64, device=x.device)
        row = table[comm.rank]
        row[0:1].copy_(n_local - n1)
        row[1:2].copy_(n1)
        row[2:2 + d].copy_(mu0)
        row[2 + d:].copy_(mu1)
        comm.allreduce_(table.view(-1))
        comm.allreduce_(S)
        check(L.dlx_gda_combine_ranks(_ptr(table), comm.world, d, _ptr(S), _ptr(n1), _ptr(mu0), _ptr(mu1),
                                      _stream()))
        return n1, mu0, mu1, S
    n1, s0, s1 = gda_pass1(x, y)
    n_total = n_local
    if comm is not None:
        comm.allreduce_(n1)
        comm.allreduce_(s0)
        comm.allreduce_(s1)
        n_total = comm.allreduce_int(n_local)
    mu0, mu1 = gda_means(n1, s0, s1, n_total)
    S = gda_pass2(x, y, mu0, mu1)
    if comm is not None:
        comm.allreduce_(S)
    return n1, mu0, mu1, S
