"""N > 1 host path on CPU: world-size-2 gloo process group.

* dist.shard partitions islands contiguously;
* the product's collective hooks (paper_1903_10741_b200.dist.make_hooks, the
  callbacks ffs_ga_config calls) implement allreduce-MAX and the rank-major
  allgather on raw pointers;
* an island GA sharded over 2 ranks, exchanging through those collectives,
  is bit-identical to the single-process run (oracle GA as the engine: the
  sharding / ring / E_max semantics are what is tested here);
* dist.global_best reduces the shards' local bests and traces to the
  single-process run's best and trace on every rank.
"""
import ctypes
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1903_10741_b200 import dist as fdist


def test_shard_partition():
    for total in (1, 2, 7, 256, 2048):
        for world in (1, 2, 3, 8):
            if world > total:
                continue
            spans = [fdist.shard(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_best(ctx, ga):
    """What ffs_best returns for a shard: its best history elite (ties ->
    lowest island), decoded, and the shard's local trace."""
    hx, hy, hobj, hfit = ga.history()
    i = int(np.argmax(hfit))
    r = ctx.decode_genes(hx[i], hy[i])
    tmin, tsum = ga.trace()
    return dict(x=hx[i], y=hy[i], assign=r["assign"], start=r["start"], objective=int(r["objective"]),
                sum_tardiness=int(r["sum_tardiness"]), makespan=int(r["makespan"]),
                trace_min=np.asarray(tmin, np.int64), trace_sum=np.asarray(tsum, np.int64))


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # --- the C-callback hooks on host memory
        allreduce, allgather = fdist.make_hooks(device_memory=False)
        v = np.array([100 + 7 * rank], dtype=np.int64)
        assert allreduce(None, v.ctypes.data, None) == 0
        assert v[0] == 100 + 7 * (world - 1)
        n = 13
        send = np.full(n, rank + 1, dtype=np.uint8)
        recv = np.zeros(n * world, dtype=np.uint8)
        assert allgather(None, send.ctypes.data, recv.ctypes.data, n, None) == 0
        assert (recv.reshape(world, n) == np.arange(1, world + 1)[:, None]).all()

        # --- sharded island GA exchanging through the same collectives
        from oracle import oracle as orc
        from paper_1903_10741_b200 import workload as wlmod
        from tests import fixtures as fx
        wl = wlmod.config_A2()
        ctx, _, _, _ = fx.oracle_event_ctx(wl)
        islands, G = 4, 22          # two migrations (k = 10, 20)
        b, e = fdist.shard(islands, rank, world)

        def ar(x):
            t = torch.tensor([x], dtype=torch.float64)
            return float(fdist.allreduce_max_tensor(t)[0])

        def ag(buf):
            t = torch.frombuffer(bytearray(buf), dtype=torch.uint8)
            return [c.numpy().tobytes() for c in fdist.allgather_bytes_tensor(t).chunk(world)]

        ga = orc.GA(ctx, 4, 2, islands, G, 4242, island_begin=b, island_end=e,
                    allreduce_max=ar, allgather=ag, rank=rank, world=world)
        for _ in range(G + 1):
            ga.step()
        x, y, obj, fit = ga.population()
        tmin, tsum = ga.trace()
        # --- the ring's global best + trace from the shards' local results
        gb = fdist.global_best(_shard_best(ctx, ga))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), x=x, y=y, obj=obj, fit=fit, tmin=tmin,
                 tsum=tsum, emax=ga.emax, gb_x=gb["x"], gb_y=gb["y"], gb_start=gb["start"],
                 gb_assign=gb["assign"], gb_obj=gb["objective"], gb_T=gb["sum_tardiness"],
                 gb_M=gb["makespan"], gb_tmin=gb["trace_min"], gb_tsum=gb["trace_sum"], gb_rank=gb["rank"])
    finally:
        dist.destroy_process_group()


def test_two_rank_island_ga_equals_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle import oracle as orc
    from paper_1903_10741_b200 import workload as wlmod
    from tests import fixtures as fx
    wl = wlmod.config_A2()
    ctx, _, _, _ = fx.oracle_event_ctx(wl)
    G = 22
    ref = orc.GA(ctx, 4, 2, 4, G, 4242)
    for _ in range(G + 1):
        ref.step()
    rx, ry, robj, rfit = ref.population()
    rmin, rsum = ref.trace()
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert (np.concatenate([p["x"] for p in parts]) == rx).all()
    assert (np.concatenate([p["y"] for p in parts]) == ry).all()
    assert (np.concatenate([p["obj"] for p in parts]) == robj).all()
    assert (np.concatenate([p["fit"] for p in parts]) == rfit).all()
    assert all(int(p["emax"]) == ref.emax for p in parts)
    # global trace = min / sum over the shards' local traces
    assert (np.minimum(parts[0]["tmin"], parts[1]["tmin"]) == rmin).all()
    assert (parts[0]["tsum"] + parts[1]["tsum"] == rsum).all()
    # dist.global_best: every rank returns the single-process run's best and trace
    ref_best = _shard_best(ctx, ref)
    for p in parts:
        assert int(p["gb_obj"]) == ref_best["objective"]
        assert int(p["gb_T"]) == ref_best["sum_tardiness"] and int(p["gb_M"]) == ref_best["makespan"]
        for k in ("x", "y", "start", "assign"):
            assert (p["gb_" + k] == ref_best[k]).all(), k
        assert (p["gb_tmin"] == rmin).all() and (p["gb_tsum"] == rsum).all()
