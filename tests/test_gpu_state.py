"""Decode-state checkpoint (louiskv_state_save / _restore) and the prefill phase timer, on the GPU."""
import numpy as np
import pytest
import torch

from synth.configs import C1, Config

from _pair import make_inputs, planted_assign, np32
import oracle

pytestmark = pytest.mark.gpu


def _lkv():
    import paper_2510_11292_b200 as lkv
    return lkv


def test_state_restore_replays_bitwise():
    """Save after 6 steps, run 10 steps, restore, run the same 10 steps again: flags, r_t, outputs,
    selections and the stats deltas are identical bit for bit (both passes through the bench's
    launch path, louiskv_decode_layer)."""
    lkv = _lkv()
    cfg = Config("st", num_layers=3, num_q_heads=8, num_kv_heads=2, head_dim=128, batch=2, prompt_len=1100,
                 decode_steps=16, sink_tokens=16, window_tokens=24, budget_tokens=96, tau=0.85,
                 avg_cluster_size=16, kmeans_iters=4, full_cache_layers=(0,), seg_mean=5.0)
    inp = make_inputs(cfg, 16, 31)
    ctx = lkv.Context(lkv.make_config(cfg))
    for l in range(cfg.num_layers):
        ctx.cluster_prompt(l, inp.K[l], inp.V[l])
    L, b, g, hn = cfg.num_layers, cfg.batch, cfg.group, cfg.num_kv_heads
    out = torch.zeros((L, b, g * hn, 128), dtype=torch.bfloat16, device="cuda")
    out32 = torch.zeros((L, b, g * hn, 128), dtype=torch.float32, device="cuda")
    fl = torch.zeros((L, b), dtype=torch.uint8, device="cuda")
    rr = torch.zeros((L, b), dtype=torch.float64, device="cuda")

    def step(t):
        for l in range(L):
            ctx.decode_layer(l, inp.q[t, l], inp.k[t, l].contiguous(), inp.v[t, l].contiguous(), out[l], out32[l],
                             fl[l], rr[l])
        torch.cuda.synchronize()
        return fl.cpu().numpy().copy(), rr.cpu().numpy().copy(), out32.cpu().numpy().copy()

    for t in range(6):
        step(t)
    ctx.state_save()
    s0 = ctx.stats()
    first = [step(t) for t in range(6, 16)]
    sel1 = [ctx.get_selection(l, bb, hh) for l in (1, 2) for bb in range(b) for hh in range(hn)]
    d1 = {k: v - s0[k] for k, v in ctx.stats().items() if not k.startswith("kmeans")}
    ctx.state_restore()
    assert ctx.stats()["retrievals"] == s0["retrievals"]
    second = [step(t) for t in range(6, 16)]
    sel2 = [ctx.get_selection(l, bb, hh) for l in (1, 2) for bb in range(b) for hh in range(hn)]
    d2 = {k: v - s0[k] for k, v in ctx.stats().items() if not k.startswith("kmeans")}
    assert sum(int(f.sum()) for f, _, _ in first) > 0
    for (f1, r1, o1), (f2, r2, o2) in zip(first, second):
        assert np.array_equal(f1, f2) and np.array_equal(r1.view(np.uint64), r2.view(np.uint64))
        assert np.array_equal(o1.view(np.uint32), o2.view(np.uint32))
    assert all(np.array_equal(a, c) for a, c in zip(sel1, sel2))
    assert d1 == d2
    ctx.close()


def test_prefill_timer_counts_and_phases():
    lkv = _lkv()
    cfg = C1.replace(kmeans_iters=5, num_kv_heads=2, num_q_heads=2, batch=2)
    inp = make_inputs(cfg, 1, 2)
    ctx = lkv.Context(lkv.make_config(cfg))
    ctx.set_prefill_timing(True)
    ctx.cluster_prompt(0, inp.K[0], inp.V[0])
    t = ctx.prefill_times()
    N, k = 4096, 64
    assert t["calls"] == 1 and t["assign_passes"] == 5 and t["keys"] == 4 * N
    assert t["assign_flops"] == 4 * N * k * 2 * 128 * 5
    assert t["d2h_bytes"] == 4 * N * 512
    for key in ("init_ms", "assign_ms", "sort_ms", "update_ms", "stage_ms", "d2h_ms"):
        assert t[key] > 0, key
    ctx.set_prefill_timing(False)
    ctx.cluster_prompt(0, inp.K[0], inp.V[0])
    assert ctx.prefill_times()["calls"] == 0
    # the clustering itself is unchanged by the timer (same units as an untimed context)
    ctx2 = lkv.Context(lkv.make_config(cfg))
    ctx2.cluster_prompt(0, inp.K[0], inp.V[0])
    for bb in range(2):
        for hh in range(2):
            c1, s1, f1 = ctx.get_units(0, bb, hh)
            c2, s2, f2 = ctx2.get_units(0, bb, hh)
            assert np.array_equal(s1, s2) and np.array_equal(c1.view(np.uint32), c2.view(np.uint32))
    ctx.close()
    ctx2.close()


def test_numa_bound_pool_path(monkeypatch):
    """The NUMA-local pool path (mmap + mbind + cudaHostRegister), forced on this single-node host:
    an episode on it matches one on the cudaHostAlloc pool bit for bit."""
    lkv = _lkv()
    cfg = Config("nu", num_layers=2, num_q_heads=8, num_kv_heads=2, head_dim=128, batch=1, prompt_len=900,
                 decode_steps=10, sink_tokens=16, window_tokens=24, budget_tokens=96, tau=0.85,
                 avg_cluster_size=16, kmeans_iters=3, full_cache_layers=(0,), seg_mean=4.0)
    inp = make_inputs(cfg, 10, 41)
    res = []
    for mode in ("1", "0"):
        monkeypatch.setenv("LOUISKV_POOL_NUMA", mode)
        ctx = lkv.Context(lkv.make_config(cfg))
        if mode == "1":
            assert ctx.pool_numa_node() >= 0
        else:
            assert ctx.pool_numa_node() == -1
        for l in range(2):
            ctx.cluster_prompt(l, inp.K[l], inp.V[l])
        out32 = torch.zeros((2, 1, 8, 128), dtype=torch.float32, device="cuda")
        out = torch.zeros((2, 1, 8, 128), dtype=torch.bfloat16, device="cuda")
        for t in range(10):
            for l in range(2):
                ctx.decode_layer(l, inp.q[t, l], inp.k[t, l].contiguous(), inp.v[t, l].contiguous(), out[l], out32[l])
        torch.cuda.synchronize()
        res.append((out32.cpu().numpy().copy(), ctx.stats(), ctx.get_working_set(1, 0, 1)))
        ctx.close()
    assert np.array_equal(res[0][0].view(np.uint32), res[1][0].view(np.uint32))
    assert res[0][1] == res[1][1] and res[0][1]["bytes_h2d"] > 0
    assert np.array_equal(res[0][2][0], res[1][2][0])
