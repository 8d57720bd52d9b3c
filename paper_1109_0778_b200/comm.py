"""Sample-sharded multi-GPU mode: NCCL allReduce of partial activation records.

One process per GPU (torchrun).  Rank 0 creates the NCCL unique id through the dlx ABI
(``dlx_comm_unique_id``), ``torch.distributed`` broadcasts it (plumbing only), and every
rank builds its dlx communicator; the per-iteration sums go through
``dlx_comm_allreduce_sum`` on the executor's stream.  Shards are contiguous sample ranges
``[r*N/G, (r+1)*N/G)``, mirroring executeDEG's contiguous chunks.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import check


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank in world (same split as the oracle's chunks)."""
    return n * rank // world, n * (rank + 1) // world


class Comm:
    def __init__(self, rank: int, world: int, uid: bytes | None = None, force_nccl: bool = False):
        """force_nccl: build the NCCL communicator even at world 1 (tests of the NCCL path)."""
        L = _lib.load()
        self.rank, self.world = rank, world
        self._h = ctypes.c_void_p()
        self._nccl = world > 1 or force_nccl
        if self._nccl:
            assert uid is not None and len(uid) == 128
            check(L.dlx_comm_init(ctypes.byref(self._h), uid, world, rank))

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(_lib.load().dlx_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls) -> "Comm":
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        return cls(rank, world, obj[0])

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if not self._nccl:
            return t
        dtype = {torch.float64: 0, torch.int64: 1}[t.dtype]
        check(_lib.load().dlx_comm_allreduce_sum(self._h, ctypes.c_void_p(t.data_ptr()), t.numel(), dtype,
                                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return t

    def allreduce_many_(self, tensors) -> None:
        """Sum several records in place across ranks with one fused NCCL launch."""
        if not self._nccl or not tensors:
            return
        n = len(tensors)
        bufs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in tensors])
        counts = (ctypes.c_int64 * n)(*[t.numel() for t in tensors])
        dtypes = (ctypes.c_int * n)(*[{torch.float64: 0, torch.int64: 1}[t.dtype] for t in tensors])
        check(_lib.load().dlx_comm_allreduce_sum_group(self._h, bufs, counts, dtypes, n,
                                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def allreduce_int(self, v: int) -> int:
        if not self._nccl:
            return v
        t = torch.tensor([v], dtype=torch.int64, device="cuda")
        self.allreduce_(t)
        return int(t.item())

    def close(self):
        if self._nccl and self._h:
            check(_lib.load().dlx_comm_destroy(self._h))
            self._h = ctypes.c_void_p()


class PeerComm:
    """Peer-memory collective (csrc/peer.cu): the partial record is summed across ranks by one
    kernel that reads every peer's exchange buffer directly (NVLink loads over NVSwitch; CUDA
    IPC within one device), folds the ranks in ascending order (bit-identical on every rank,
    SPEC.md:648's ascending-chunk combine lifted to ranks) and applies the update that consumes
    the sum in the same launch.  The exchange buffers' IPC handles travel once through
    ``torch.distributed`` (any backend: plumbing only).  Same interface as :class:`Comm`, plus
    the fused ``kmeans_update_`` / ``bgd_step_``."""

    HANDLE_BYTES = 64

    def __init__(self, rank: int, world: int, cap_bytes: int = 8 << 20, group=None):
        L = _lib.load()
        self.rank, self.world, self.cap = rank, world, int(cap_bytes)
        self._own = ctypes.c_void_p()
        h = ctypes.create_string_buffer(self.HANDLE_BYTES)
        check(L.dlx_peer_alloc(self.cap, ctypes.byref(self._own), h))
        handles = [h.raw]
        if world > 1:
            import torch.distributed as dist
            handles = [None] * world
            dist.all_gather_object(handles, h.raw, group=group)
        self._opened = []
        ptrs = []
        for q in range(world):
            if q == rank:
                ptrs.append(self._own.value)
                continue
            p = ctypes.c_void_p()
            check(L.dlx_peer_open(handles[q], ctypes.byref(p)))
            self._opened.append(p)
            ptrs.append(p.value)
        self._bufs = (ctypes.c_void_p * world)(*ptrs)

    @classmethod
    def from_torch_distributed(cls, cap_bytes: int = 8 << 20) -> "PeerComm":
        import torch.distributed as dist
        return cls(dist.get_rank(), dist.get_world_size(), cap_bytes)

    def _run(self, items, ni, nf, counts, sums, epilogue=0, out=None, alpha=0.0):
        ptr = lambda t: ctypes.c_void_p(t.data_ptr() if t is not None else None)  # noqa: E731
        check(_lib.load().dlx_peer_allreduce(
            self._bufs, self.world, self.rank, self.cap, int(items), int(ni), int(nf),
            ptr(counts), ptr(sums), int(epilogue), ptr(out), float(alpha),
            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        assert t.is_contiguous() and t.dtype in (torch.float64, torch.int64)
        if t.dtype == torch.int64:
            self._run(t.numel(), 1, 0, t, None)
        else:
            self._run(t.numel(), 0, 1, None, t)
        return t

    def allreduce_many_(self, tensors) -> None:
        for t in tensors:
            self.allreduce_(t)

    def allreduce_int(self, v: int) -> int:
        t = torch.tensor([v], dtype=torch.int64, device="cuda")
        self.allreduce_(t)
        return int(t.item())

    def kmeans_update_(self, counts: torch.Tensor, sums: torch.Tensor, mu: torch.Tensor) -> None:
        """counts (k,) int64 and sums (k, d) fp64 summed across ranks in place, then
        mu = sums / toDouble(counts) (kmeans_update's semantics), in one launch."""
        k, d = sums.shape
        self._run(k, 1, d, counts, sums, epilogue=1, out=mu)

    def bgd_step_(self, grad: torch.Tensor, theta: torch.Tensor, alpha: float) -> None:
        """grad summed across ranks in place, then theta -= alpha * grad (axpy_inplace)."""
        self._run(grad.numel(), 0, 1, None, grad, epilogue=2, out=theta, alpha=alpha)

    def close(self):
        L = _lib.load()
        for p in self._opened:
            check(L.dlx_peer_close(p))
        self._opened = []
        if self._own:
            check(L.dlx_peer_free(self._own))
            self._own = ctypes.c_void_p()
