"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL) for the collectives.

The path shards by contiguous column blocks (the paper's node partitioning,
PAPER.md:55): rank r owns blocks [r·G/P, (r+1)·G/P) and the matching columns of A.
The C library never talks to NCCL itself — it calls back into the host through
``bcur_comm.allreduce_f64`` (an in-place fp64 sum of a device buffer, enqueued on the
library's stream); this module provides that callback over torch.distributed, plus
the shard arithmetic shared by bench.py and the tests.  With a CPU (gloo) group the
callback also accepts host buffers, which is how the multi-rank host logic is tested
without GPUs.
"""
from __future__ import annotations

import ctypes
from typing import Callable, Optional, Tuple

import numpy as np


def block_range(G: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block range [g0, g1) of ``rank`` (remainder blocks go to the first ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("block_range: need 0 <= rank < world")
    if G < world:
        raise ValueError(f"block_range: {G} blocks cannot be split over {world} ranks")
    q, r = divmod(G, world)
    g0 = rank * q + min(rank, r)
    return g0, g0 + q + (1 if rank < r else 0)


def shard_columns(offsets, rank: int, world: int) -> Tuple[int, int, int, int]:
    """Column shard of ``rank`` for a partition given by its G+1 offsets:
    (col0, n_local, g0, g1)."""
    off = np.asarray(offsets, dtype=np.int64)
    g0, g1 = block_range(len(off) - 1, rank, world)
    return int(off[g0]), int(off[g1] - off[g0]), g0, g1


def torch_allreduce(device: str = "cuda", group=None) -> Callable[[int, int, int], None]:
    """The ``bcur_comm`` callback over torch.distributed: in-place sum of ``count``
    doubles at ``ptr``.  device="cuda": ptr is device memory and the reduction is
    enqueued on the library's stream; device="cpu": ptr is host memory (gloo)."""
    import torch
    import torch.distributed as dist

    if device == "cpu":
        def allreduce(ptr: int, count: int, stream: int) -> None:
            buf = (ctypes.c_double * count).from_address(ptr)
            t = torch.from_numpy(np.frombuffer(buf, dtype=np.float64))
            dist.all_reduce(t, group=group)
        return allreduce

    dev = torch.device(device) if device != "cuda" else torch.device("cuda", torch.cuda.current_device())

    class _Cai:
        def __init__(self, ptr, count):
            self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False),
                                             "version": 3, "strides": None}

    def allreduce(ptr: int, count: int, stream: int) -> None:
        t = torch.as_tensor(_Cai(ptr, count), device=dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            dist.all_reduce(t, group=group)

    return allreduce


def torch_broadcast(device: str = "cuda", group=None) -> Callable[[int, int, int, int], None]:
    """The ``bcur_comm.broadcast`` callback over torch.distributed: ``nbytes`` bytes at
    ``ptr`` from rank ``root``, in place (device memory on the library's stream, or host
    memory with a CPU/gloo group)."""
    import torch
    import torch.distributed as dist

    if device == "cpu":
        def broadcast(ptr: int, nbytes: int, root: int, stream: int) -> None:
            buf = (ctypes.c_uint8 * nbytes).from_address(ptr)
            t = torch.from_numpy(np.frombuffer(buf, dtype=np.uint8))
            dist.broadcast(t, src=root, group=group)
        return broadcast

    dev = torch.device(device) if device != "cuda" else torch.device("cuda", torch.cuda.current_device())

    class _Cai:
        def __init__(self, ptr, nbytes):
            self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                             "version": 3, "strides": None}

    def broadcast(ptr: int, nbytes: int, root: int, stream: int) -> None:
        t = torch.as_tensor(_Cai(ptr, nbytes), device=dev)
        with torch.cuda.stream(torch.cuda.ExternalStream(stream, device=dev)):
            dist.broadcast(t, src=root, group=group)

    return broadcast


def attach(ctx, rank: int, world: int, device: str = "cuda", group=None) -> None:
    """Install the torch.distributed callbacks on a bcur Context (world 1 → detach)."""
    if world <= 1:
        ctx.set_comm(0, 1, None)
        return
    ctx.set_comm(rank, world, torch_allreduce(device, group), torch_broadcast(device, group))


def max_over_ranks(value: float, device: Optional[str] = None) -> float:
    """Max of a per-rank scalar (bench timing: the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device or "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
