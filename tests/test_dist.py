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
    # the per-step batched variant (--gather step): one all-gather of [L, b, g*hc, d]
    L = 3
    full_s = torch.arange(L * b * Hq * d, dtype=torch.float32).reshape(L, b, Hq, d)
    own_s = full_s[:, :, hb * g:(hb + hc) * g].contiguous()
    gathered_s = torch.empty((world, L, b, g * hc, d), dtype=torch.float32)
    bench.gather_heads(own_s, gathered_s, world)
    ok = ok and torch.equal(bench.assemble_heads(gathered_s), full_s)
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


def _oracle_heads_worker(rank, world, port, out):
    """Rank r runs the ORACLE decode for its KV-head shard (the decomposition the GPU ranks use:
    every rank sees all query heads for the trigger, and only its heads' KV); the per-layer
    outputs go through gather_heads / assemble_heads (gloo)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import torch
    import torch.distributed as dist
    import bench
    import synth
    from synth.configs import Config
    from oracle.episode import OracleEpisode
    from _pair import planted_assign
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = Config("d", num_layers=2, num_q_heads=8, num_kv_heads=4, head_dim=128, batch=2, prompt_len=300,
                 decode_steps=6, sink_tokens=8, window_tokens=16, budget_tokens=48, tau=0.85, avg_cluster_size=16,
                 kmeans_iters=2, full_cache_layers=(0,), seg_mean=3.0)
    hb, hc = bench.head_range(rank, world, cfg.num_kv_heads)
    plants = [synth.planted(cfg, l, 3, "cpu") for l in range(2)]
    KV = [synth.prompt_kv(cfg, l, 3, "cpu", plants[l], return_labels=True) for l in range(2)]
    q, k, v, _ = synth.decode_stream(cfg, 6, 3, "cpu", plants)
    ep = OracleEpisode(cfg, kv_head_begin=hb, kv_head_count=hc)
    for l in range(2):
        K, V, lab = KV[l]
        Kn, Vn = K[:, :, hb:hb + hc].float().numpy(), V[:, :, hb:hb + hc].float().numpy()
        if l == 0:
            ep.cluster_prompt(l, Kn, Vn)
        else:
            ep.cluster_prompt(l, Kn, Vn, assign=planted_assign(cfg, lab[:, :, hb:hb + hc]))
    outs = []
    g = cfg.group
    for t in range(6):
        for l in range(2):
            qa = q[t, l].float().numpy()
            ep.should_retrieve(l, qa)
            qo = qa[:, hb * g:(hb + hc) * g]
            ep.retrieve(l, qo)
            ep.append_output(l, k[t, l][:, hb:hb + hc].float().numpy(), v[t, l][:, hb:hb + hc].float().numpy())
            own = torch.from_numpy(ep.sparse_attn(l, qo))
            gathered = torch.empty((world,) + tuple(own.shape), dtype=own.dtype)
            bench.gather_heads(own.contiguous(), gathered, world)
            outs.append(bench.assemble_heads(gathered).numpy())
    out.put((rank, np.stack(outs)))
    dist.destroy_process_group()


def test_oracle_head_shards_all_gather_equal_full_run_gloo():
    """north_star's multi-GPU decomposition, checked on CPU: two ranks each run the oracle on half the
    KV heads; the all-gathered, assembled outputs of every layer and step equal the single-process
    oracle run over all heads bit for bit (no cross-rank arithmetic)."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import synth
    from synth.configs import Config
    from oracle.episode import OracleEpisode
    from _pair import planted_assign
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_heads_worker, args=(r, 2, port, q_)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q_.get(timeout=300) for _ in range(2)), key=lambda z: z[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = Config("d", num_layers=2, num_q_heads=8, num_kv_heads=4, head_dim=128, batch=2, prompt_len=300,
                 decode_steps=6, sink_tokens=8, window_tokens=16, budget_tokens=48, tau=0.85, avg_cluster_size=16,
                 kmeans_iters=2, full_cache_layers=(0,), seg_mean=3.0)
    plants = [synth.planted(cfg, l, 3, "cpu") for l in range(2)]
    KV = [synth.prompt_kv(cfg, l, 3, "cpu", plants[l], return_labels=True) for l in range(2)]
    q, k, v, _ = synth.decode_stream(cfg, 6, 3, "cpu", plants)
    ep = OracleEpisode(cfg)
    for l in range(2):
        K, V, lab = KV[l]
        if l == 0:
            ep.cluster_prompt(l, K.float().numpy(), V.float().numpy())
        else:
            ep.cluster_prompt(l, K.float().numpy(), V.float().numpy(), assign=planted_assign(cfg, lab))
    ref = []
    for t in range(6):
        for l in range(2):
            qa = q[t, l].float().numpy()
            ep.should_retrieve(l, qa)
            ep.retrieve(l, qa)
            ep.append_output(l, k[t, l].float().numpy(), v[t, l].float().numpy())
            ref.append(ep.sparse_attn(l, qa))
    ref = np.stack(ref)
    assert ep.stats["retrievals"] > 0
    for r, arr in res:
        assert np.array_equal(arr, ref), r
