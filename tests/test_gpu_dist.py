"""The sharded island GA through the C-ABI's collective hooks on the GPU:
two processes (gloo; both on cuda:0, since this box has one GPU), each owning
half of the islands, exchanging E_max and the ring migrants through the
callbacks of ffs_ga_config -- bit-identical to the single-process run (every
random draw is keyed by the global island index; R22, R23)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ISL_W, ISL_H, ISLANDS, G, SEED = 4, 4, 6, 23, 31


def _state():
    from paper_1903_10741_b200 import ffs
    from paper_1903_10741_b200 import workload as wlmod
    wl = wlmod.config_A2()
    base = ffs.Instance.from_arrays(wl.original_instance(), device=0)
    st0 = ffs.make_state(base, 0)
    assign, start, _, _, M = ffs.decode_schedule(st0, wl.plan_x, wl.plan_y)
    rs = wl.rs_from_makespan(wl.ratios[0], M)
    inst = ffs.Instance.from_arrays(wl.instance_at(0, [rs]), device=0)
    st = ffs.make_state(inst, rs, assign[: wl.n * wl.g], start[: wl.n * wl.g])
    st._keep = (base, st0, inst)
    return st


def _state_c():
    """Config C's frozen state (K = 855), built on the GPU as bench.py does."""
    from paper_1903_10741_b200 import ffs
    from paper_1903_10741_b200 import workload as wlmod
    wl = wlmod.config_C()
    base = ffs.Instance.from_arrays(wl.original_instance(), device=0)
    st0 = ffs.make_state(base, 0)
    assign, start, _, _, M = ffs.decode_schedule(st0, wl.plan_x, wl.plan_y)
    rs = wl.rs_from_makespan(wl.ratios[0], M)
    inst = ffs.Instance.from_arrays(wl.instance_at(0, [rs]), device=0)
    st = ffs.make_state(inst, rs, wl.plan_x.astype(np.int32), start[: wl.n * wl.g])
    st._keep = (base, st0, inst)
    return st


def _worker(rank, world, port, out_dir, cfg="A"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_10741_b200 import dist as fdist
        from paper_1903_10741_b200 import ffs
        torch.cuda.set_device(0)
        st, (w, h, isl, g, mi) = (_state(), (ISL_W, ISL_H, ISLANDS, G, 10)) if cfg == "A" else (_state_c(), C_SHAPE)
        b, e = fdist.shard(isl, rank, world)
        run = ffs.Run(st, w, h, isl, g, SEED, island_begin=b, island_end=e, rank=rank, world=world,
                      hooks=fdist.make_hooks(device_memory=True), migration_interval=mi)
        run.step(g)
        x, y, obj, fit = run.population()
        hx, hy, hobj, hfit = run.history()
        gb = fdist.global_best(run.best())
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=x, y=y, obj=obj, fit=fit, hx=hx, hy=hy, hobj=hobj,
                 emax=run.info()["emax"], **{"gb_" + k: np.asarray(v) for k, v in gb.items()})
    finally:
        dist.destroy_process_group()


C_SHAPE = (16, 16, 6, 9, 4)   # config C tiles, 6 islands over 2 ranks, 9 generations, migration every 4


@pytest.mark.parametrize("cfg,world", [("A", 2), ("C", 2), ("A", 3), ("A", 4)])
def test_two_rank_ga_equals_single_process(tmp_path, cfg, world):
    """cfg C: config C's instance (K = 855: 2,581-byte migration records) in
    16x16 tiles, the ring crossing the shard boundary in both migrations.
    world 3 / 4: uneven and one-island shards (6 islands), the ring's
    wrap-around import (rank 0 <- the last rank) through the allgather."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(world, port, str(tmp_path), cfg), nprocs=world, join=True)
    from paper_1903_10741_b200 import ffs
    st, (w, h, isl, g, mi) = (_state(), (ISL_W, ISL_H, ISLANDS, G, 10)) if cfg == "A" else (_state_c(), C_SHAPE)
    run = ffs.Run(st, w, h, isl, g, SEED, migration_interval=mi)
    run.step(g)
    x, y, obj, fit = run.population()
    hx, hy, hobj, _ = run.history()
    parts = [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]
    assert all(int(p["emax"]) == run.info()["emax"] for p in parts)
    for key, ref in (("x", x), ("y", y), ("obj", obj), ("fit", fit), ("hx", hx), ("hy", hy), ("hobj", hobj)):
        got = np.concatenate([p[key] for p in parts])
        assert (got == ref).all(), key
    # the ring's global best and trace (dist.global_best) on every rank == the single run's ffs_best
    b = run.best()
    for p in parts:
        for k in ("x", "y", "assign", "start", "trace_min", "trace_sum", "objective", "sum_tardiness", "makespan"):
            assert (p["gb_" + k] == np.asarray(b[k])).all(), k


def _nccl_worker(rank, world, port, out_dir):
    """World-1 NCCL group on the GPU: the product's hooks (make_hooks with
    device memory) called on raw device pointers and the library's stream
    handle (ExternalStream), then global_best over NCCL."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        from paper_1903_10741_b200 import dist as fdist
        from paper_1903_10741_b200 import ffs
        allreduce, allgather = fdist.make_hooks(device_memory=True)
        s = torch.cuda.Stream()
        v = torch.tensor([12345], dtype=torch.int64, device="cuda")
        send = torch.arange(40, dtype=torch.uint8, device="cuda")
        recv = torch.zeros(40 * world, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        assert allreduce(None, v.data_ptr(), s.cuda_stream) == 0
        assert allgather(None, send.data_ptr(), recv.data_ptr(), 40, s.cuda_stream) == 0
        s.synchronize()
        assert int(v.item()) == 12345 and bool((recv == send).all())
        st = _state()
        run = ffs.Run(st, ISL_W, ISL_H, ISLANDS, 12, SEED, stream=s)
        run.step(12)
        gb = fdist.global_best(run.best())
        b = run.best()
        ok = all(bool((np.asarray(gb[k]) == np.asarray(b[k])).all())
                 for k in ("x", "y", "start", "trace_min", "trace_sum", "objective"))
        open(os.path.join(out_dir, "nccl_ok"), "w").write(f"{ok} {dist.get_backend()}")
    finally:
        dist.destroy_process_group()


def test_nccl_hooks_world_one(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_nccl_worker, args=(1, port, str(tmp_path)), nprocs=1, join=True)
    assert open(os.path.join(tmp_path, "nccl_ok")).read() == "True nccl"


def test_bench_two_ranks_under_torchrun():
    """bench.py's multi-GPU launch (torchrun, one process per rank, barrier +
    max-over-ranks timing, global best of the ring) with two ranks sharing
    cuda:0 over gloo (this box has one GPU; NCCL refuses two ranks on one
    device): rank 0 prints one JSON line for the whole 2 x 256-island job."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, FFS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["config"]["islands_total"] == 512 and d["config"]["population_total"] == 2 * 65536
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["value"] == pytest.approx(2 * 65536 * 3 / (d["ms_per_step"] * 3e-3), rel=1e-6)
