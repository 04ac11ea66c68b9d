"""Row sharding over the GPUs of one node.

Rows of C and X are split contiguously, ``row_range(m)`` =
[rank*m/W, (rank+1)*m/W); every row-local quantity (lse, zeta, CSR rows,
z_i, e_r) stays on its rank.  The length-n vectors (gradient, d = P_rho^T a,
the H v product of every CG iteration, the rounding column sums, the
warm-start column statistics) are combined by NCCL all-reduce inside
libotb, on the solver's stream; the n-dimensional Newton/CG state is
replicated, and because every rank reduces the same all-reduced values in
the same order, every rank takes the same control-flow decisions without
further communication.

``RowComm`` is the plumbing: it takes ranks from ``torch.distributed``
(one process per GPU), creates the NCCL unique id on rank 0 and broadcasts
its 128 bytes over the default process group (gloo or nccl), then attaches
a communicator to each rank's libotb context.  The row partition and the
id exchange are pure host logic and are tested with gloo on the CPU.
"""

from __future__ import annotations

import ctypes as C


def row_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced row shard of rank ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * m) // world, ((rank + 1) * m) // world


def anchor_owner(anchor: int, m: int, world: int) -> int:
    """Rank whose shard holds the global anchor row."""
    for r in range(world):
        lo, hi = row_range(m, r, world)
        if lo <= anchor < hi:
            return r
    raise ValueError("anchor out of range")


def broadcast_id(payload: bytes | None, group=None) -> bytes:
    """Broadcast rank 0's 128-byte NCCL id to every rank (torch.distributed)."""
    import torch.distributed as dist

    obj = [payload]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class RowComm:
    """Rank / world of torch.distributed plus the NCCL attach for libotb."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def row_range(self, m: int) -> tuple[int, int]:
        return row_range(m, self.rank, self.world)

    def attach(self, session) -> None:
        if self.world == 1:
            return
        from . import _lib

        path = _lib.nccl_path().encode()
        uid = None
        if self.rank == 0:
            buf = (C.c_char * 128)()
            _lib.check(_lib.lib.otb_nccl_get_unique_id(path, buf))
            uid = bytes(buf)
        uid = broadcast_id(uid, self.group)
        raw = (C.c_char * 128).from_buffer_copy(uid)
        _lib.check(_lib.lib.otb_attach_nccl(session.ctx, path, raw, self.world, self.rank))
