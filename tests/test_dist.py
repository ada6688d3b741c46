"""world_size-2 CPU (gloo) tests of the multi-rank host logic used by bench.py."""
import os
import socket
import subprocess
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = bench.max_over_ranks(10.0 * (rank + 1), world)
    dist.barrier()
    out.put((rank, m, bench.rank_seed(7, rank)))
    dist.destroy_process_group()


def test_max_over_ranks_and_independent_seeds_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [20.0, 20.0]          # max over ranks, seen by every rank
    assert res[0][2] != res[1][2]                       # weak scaling: independent problems


def test_reference_arm_rank1_exits_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == ""


def _heads_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, Hq, Hkv, d = 3, 32, 8, 16
    g = Hq // Hkv
    full = torch.arange(b * Hq * d, dtype=torch.float32).reshape(b, Hq, d)  # "attention output" of every head
    hb, hc = bench.head_range(rank, world, Hkv)
    own = full[:, hb * g:(hb + hc) * g].contiguous()  # what this rank's ctx computes (its KV heads' groups)
    gathered = torch.empty((world, b, g * hc, d), dtype=torch.float32)
    bench.gather_heads(own, gathered, world)
    ok = torch.equal(bench.assemble_heads(gathered), full)
    out.put((rank, hb, hc, ok))
    dist.destroy_process_group()


def test_head_shard_all_gather_assembles_model_head_order_gloo():
    """--shard heads: contiguous KV-head ranges, and the per-layer all-gather + assembly returns every
    query head's output in model order (q head h belongs to KV head h // g)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_heads_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 4), (4, 4)]
    assert all(r[3] for r in res)


def test_head_range_rejects_uneven_split():
    sys.path.insert(0, ROOT)
    import bench
    import pytest
    with pytest.raises(ValueError):
        bench.head_range(0, 3, 8)
    assert [bench.head_range(r, 8, 8) for r in range(8)] == [(r, 1) for r in range(8)]
