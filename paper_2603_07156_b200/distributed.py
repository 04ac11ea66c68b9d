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

``LocalGroup`` runs the same sharded path inside ONE process: ``world``
host threads, one libotb context each (all on one GPU in the tests), whose
all-reduces are a fixed-order device sum of the ranks' buffers
(otb_attach_group, include/otb.h).  Every collective call site of the NCCL
path runs unchanged, so a single-GPU box checks the sharded reductions of
semidual.py:98-100 (gradient), sparsify.py:143-153 (d, H v),
feasibility.py:56-66 (rounding column sums) and sinkhorn.py:54-58 (the
gamma sweep) against the one-rank result (tests/test_gpu_multirank.py).
"""

from __future__ import annotations

import ctypes as C
import os
import threading


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

    def all_reduce_(self, t, op: str = "sum"):
        """In-place all-reduce of a torch tensor over the process group."""
        if self.world == 1:
            return t
        import torch.distributed as dist

        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM, group=self.group)
        return t

    def attach(self, session) -> None:
        # OTB_NCCL_SELFTEST=1: a one-rank communicator is attached too and the
        # context runs every multi-rank code path (otb_attach_nccl), so a
        # one-GPU box exercises the NCCL binding
        if self.world == 1 and os.environ.get("OTB_NCCL_SELFTEST") != "1":
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


class LocalGroup:
    """``world`` ranks of one process (one host thread per rank) sharing a
    libotb local group.  ``comm(rank)`` is the rank's communicator, used
    exactly like ``RowComm`` (``ibsn_solve(..., comm=...)``)."""

    def __init__(self, world: int):
        from . import _lib

        if world < 1:
            raise ValueError("world must be >= 1")
        self.world = world
        self.handle = C.c_void_p()
        _lib.check(_lib.lib.otb_group_create(C.byref(self.handle), world))
        self._barrier = threading.Barrier(world)
        self._slots: list = [None] * world
        self._comms = [LocalComm(self, r) for r in range(world)]

    def comm(self, rank: int) -> "LocalComm":
        return self._comms[rank]

    def abort(self) -> None:
        from . import _lib

        self._barrier.abort()
        if self.handle:
            _lib.lib.otb_group_abort(self.handle)

    def close(self) -> None:
        from . import _lib

        if self.handle:
            _lib.lib.otb_group_destroy(self.handle)
            self.handle = C.c_void_p()

    def run(self, fn, *, timeout: float = 600.0):
        """Run ``fn(rank, comm)`` on ``world`` threads, each on its own CUDA
        stream; returns the per-rank results.  The first exception aborts
        the group (the other ranks fail out of their barriers) and is
        re-raised."""
        import torch

        results: list = [None] * self.world
        errors: list = []          # in the order they were raised
        lock = threading.Lock()
        dev = torch.cuda.current_device()

        def body(r):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(torch.cuda.Stream(dev)):
                    results[r] = fn(r, self._comms[r])
                    torch.cuda.current_stream().synchronize()
            except BaseException as e:   # noqa: BLE001 - re-raised below
                with lock:
                    errors.append(e)
                self.abort()

        threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout)
        if any(t.is_alive() for t in threads):
            self.abort()
            raise TimeoutError("local group ranks did not finish")
        if errors:
            raise errors[0]   # the first failure; the others are its consequences
        return results


class LocalComm:
    """One rank of a LocalGroup (duck-types RowComm)."""

    def __init__(self, group: LocalGroup, rank: int):
        self._g = group
        self.rank = rank
        self.world = group.world

    def row_range(self, m: int) -> tuple[int, int]:
        return row_range(m, self.rank, self.world)

    def all_reduce_(self, t, op: str = "sum"):
        """In-place all-reduce of a device tensor across the group's threads
        (rank-ordered sum / max; set-up scalars only, host-synchronised)."""
        if self.world == 1:
            return t
        import torch

        g = self._g
        torch.cuda.current_stream(t.device).synchronize()
        g._slots[self.rank] = t
        g._barrier.wait()
        acc = g._slots[0].clone()
        for q in range(1, self.world):
            acc = torch.maximum(acc, g._slots[q]) if op == "max" else acc + g._slots[q]
        torch.cuda.current_stream(t.device).synchronize()
        g._barrier.wait()
        t.copy_(acc)
        return t

    def attach(self, session) -> None:
        from . import _lib

        _lib.check(_lib.lib.otb_attach_group(session.ctx, self._g.handle, self.rank))
