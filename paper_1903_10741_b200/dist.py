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


def global_best(best: dict) -> dict:
    """The ring's result from every shard's ffs_best.

    The answer of the island GA is the best individual in history over all
    islands and the trace is over the whole population
    (S:199-202); each rank's `Run.best()` covers its own shard only.  One
    allgather (rank-major) of each shard's record -- objective word, sum T,
    C_max, x, y, merged schedule, local trace -- then, identically on every
    rank: the best is the smallest objective (fitness Eq. (13) is strictly
    decreasing in it above 0), ties -> lowest rank, which holds the lowest
    global islands (shards are contiguous, ties -> lowest island, R28);
    trace_min = min over shards, trace_sum = sum over shards in rank order
    (exact for the integer objective).  Returns Run.best()'s keys plus
    "rank" (the shard that holds it).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    real = isinstance(best["objective"], float)
    K = best["x"].size
    cells = best["start"].size
    G1 = best["trace_min"].size

    def word(v):
        return int(np.array([v], np.float64).view(np.int64)[0]) if real else int(v)

    head = np.array([word(best["objective"]), best["sum_tardiness"], best["makespan"]], np.int64)
    tmin = np.asarray(best["trace_min"])
    tsum = np.asarray(best["trace_sum"])
    if real:
        tmin, tsum = tmin.astype(np.float64).view(np.int64), tsum.astype(np.float64).view(np.int64)
    parts = [head, tmin.astype(np.int64), tsum.astype(np.int64)]
    rec = b"".join([p.tobytes() for p in parts] + [np.asarray(best["x"], np.int8).tobytes(),
                                                   np.asarray(best["y"], np.int16).tobytes(),
                                                   np.asarray(best["assign"], np.int32).tobytes(),
                                                   np.asarray(best["start"], np.int32).tobytes()])
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    send = torch.frombuffer(bytearray(rec), dtype=torch.uint8).to(dev)
    allb = allgather_bytes_tensor(send).cpu().numpy().reshape(world, len(rec))
    n64 = 3 + 2 * G1

    def unpack(r):
        b = allb[r]
        v = b[: 8 * n64].view(np.int64)
        o = 8 * n64
        x = b[o:o + K].view(np.int8); o += K
        y = b[o:o + 2 * K].view(np.int16); o += 2 * K
        a = b[o:o + 4 * cells].view(np.int32); o += 4 * cells
        s = b[o:o + 4 * cells].view(np.int32)
        return v[:3], v[3:3 + G1], v[3 + G1:], x, y, a, s

    recs = [unpack(r) for r in range(world)]
    r = min(range(world), key=lambda i: (int(recs[i][0][0]), i))
    head, _, _, x, y, a, s = recs[r]
    tmin_all = np.stack([q[1] for q in recs])
    tsum_all = np.stack([q[2] for q in recs])
    if real:
        obj = float(head[:1].view(np.float64)[0])
        gmin = tmin_all.min(axis=0).view(np.float64)
        gsum = np.zeros(G1, np.float64)
        for q in tsum_all.view(np.float64):       # rank order
            gsum = gsum + q
    else:
        obj = int(head[0])
        gmin = tmin_all.min(axis=0)
        gsum = tsum_all.sum(axis=0)
    return dict(x=x.copy(), y=y.copy(), assign=a.copy(), start=s.copy(), objective=obj,
                sum_tardiness=int(head[1]), makespan=int(head[2]), trace_min=gmin, trace_sum=gsum, rank=r)
