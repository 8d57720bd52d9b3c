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
    def __init__(self, rank: int, world: int, uid: bytes | None = None):
        L = _lib.load()
        self.rank, self.world = rank, world
        self._h = ctypes.c_void_p()
        if world > 1:
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
        if self.world == 1:
            return t
        dtype = {torch.float64: 0, torch.int64: 1}[t.dtype]
        check(_lib.load().dlx_comm_allreduce_sum(self._h, ctypes.c_void_p(t.data_ptr()), t.numel(), dtype,
                                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return t

    def allreduce_many_(self, tensors) -> None:
        """Sum several records in place across ranks with one fused NCCL launch."""
        if self.world == 1 or not tensors:
            return
        n = len(tensors)
        bufs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in tensors])
        counts = (ctypes.c_int64 * n)(*[t.numel() for t in tensors])
        dtypes = (ctypes.c_int * n)(*[{torch.float64: 0, torch.int64: 1}[t.dtype] for t in tensors])
        check(_lib.load().dlx_comm_allreduce_sum_group(self._h, bufs, counts, dtypes, n,
                                                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def allreduce_int(self, v: int) -> int:
        if self.world == 1:
            return v
        t = torch.tensor([v], dtype=torch.int64, device="cuda")
        self.allreduce_(t)
        return int(t.item())

    def close(self):
        if self.world > 1 and self._h:
            check(_lib.load().dlx_comm_destroy(self._h))
            self._h = ctypes.c_void_p()
