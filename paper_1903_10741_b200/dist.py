"""Island sharding over processes with torch.distributed (NCCL on GPUs, gloo
in the CPU tests): the collective hooks of ffs_ga_config.

Islands shard naturally (islands are independent between migrations);
the only exchanges are one allreduce-MAX of the initial objective (E_max over
the global population, reading R23) and, every migration_interval
generations, an allgather of each shard's boundary elite (single-ring
migration): shard r's first island receives the best of global island
r*L - 1, the last island of shard r-1 (mod W).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def shard(islands_total: int, rank: int, world: int):
    """[begin, end) global islands of `rank` (contiguous blocks, sizes differ by <= 1)."""
    base, rem = divmod(islands_total, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def allreduce_max_tensor(t):
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t


def allgather_bytes_tensor(send):
    """Gather a uint8 tensor of equal size from every rank (rank-major)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    out = torch.empty(world * send.numel(), dtype=send.dtype, device=send.device)
    if send.is_cuda:
        dist.all_gather_into_tensor(out, send)
    else:
        dist.all_gather(list(out.chunk(world)), send)
    return out


class _CAI:
    """Minimal __cuda_array_interface__ view of a raw device pointer."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _dev_view(ptr: int, n: int, typestr: str):
    import torch
    return torch.as_tensor(_CAI(ptr, n, typestr), device="cuda")


def _host_view(ptr: int, n: int, ctype):
    import torch
    return torch.from_numpy(np.ctypeslib.as_array((ctype * n).from_address(ptr)))


def make_hooks(device_memory: bool = True):
    """(allreduce_max_i64, allgather) callables for ffs.Run(hooks=...).

    device_memory=True: pointers are CUDA device pointers and `stream` is the
    cudaStream_t the library is issuing on (the collectives are ordered on it).
    """
    import torch

    def _stream_ctx(stream):
        if device_memory and stream:
            return torch.cuda.stream(torch.cuda.ExternalStream(stream))
        import contextlib
        return contextlib.nullcontext()

    def _host_staged():
        # gloo moves host tensors: device buffers are staged through the host
        # (NCCL, the GPU path, reads and writes them in place)
        import torch.distributed as dist
        return device_memory and dist.get_backend() == "gloo"

    def allreduce(user, ptr, stream):
        try:
            with _stream_ctx(stream):
                t = _dev_view(ptr, 1, "<i8") if device_memory else _host_view(ptr, 1, C.c_int64)
                if _host_staged():
                    h = t.cpu()
                    allreduce_max_tensor(h)
                    t.copy_(h)
                else:
                    allreduce_max_tensor(t)
            return 0
        except Exception:  # the C side turns non-zero into FFS_ERR_COMM
            return 1

    def allgather(user, send, recv, nbytes, stream):
        try:
            import torch.distributed as dist
            world = dist.get_world_size()
            with _stream_ctx(stream):
                if device_memory:
                    s = _dev_view(send, nbytes, "|u1")
                    r = _dev_view(recv, nbytes * world, "|u1")
                    if _host_staged():
                        r.copy_(allgather_bytes_tensor(s.cpu()))
                    else:
                        dist.all_gather_into_tensor(r, s)
                else:
                    s = _host_view(send, nbytes, C.c_uint8)
                    r = _host_view(recv, nbytes * world, C.c_uint8)
                    r.copy_(allgather_bytes_tensor(s))
            return 0
        except Exception:
            return 1

    return allreduce, allgather
