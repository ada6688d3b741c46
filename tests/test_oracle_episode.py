"""Pins for the oracle's Algorithm-1 episode: segmentation,
eviction, degeneracies, coverage and the superset-budget identity."""
import numpy as np
import pytest

import oracle
import synth
from oracle.episode import OracleEpisode, LAST_RETRIEVAL, PREV_STEP, SHARED
from synth.configs import Config


def tiny_cfg(**kw):
    base = dict(name="tiny", num_layers=1, num_q_heads=2, num_kv_heads=1, head_dim=16, batch=1,
                prompt_len=64, decode_steps=24, sink_tokens=4, window_tokens=12, budget_tokens=16,
                tau=0.5, avg_cluster_size=8, kmeans_iters=4, full_cache_layers=())
    base.update(kw)
    return Config(**base)


def _prompt(cfg, seed=0):
    rng = np.random.default_rng(seed)
    K = oracle.bf16_round(rng.standard_normal((cfg.batch, cfg.prompt_len, cfg.num_kv_heads, cfg.head_dim)).astype(np.float32))
    V = oracle.bf16_round(rng.standard_normal(K.shape).astype(np.float32))
    return K, V


def _controlled_queries(cfg, boundary_steps, seed=1):
    """q constant within a segment, a fresh orthogonal-ish direction at each boundary."""
    rng = np.random.default_rng(seed)
    T, d, H = cfg.decode_steps, cfg.head_dim, cfg.num_q_heads
    q = np.zeros((T, cfg.num_layers, cfg.batch, H, d), np.float32)
    cur = None
    for t in range(1, T + 1):
        if t in boundary_steps or cur is None:
            cur = np.zeros((H, d), np.float32)
            cur[:, (t * 3) % d] = 1.0  # one-hot: cosine 0 across boundaries, 1 within
        q[t - 1, :, :] = cur
    k = oracle.bf16_round(rng.standard_normal((T, cfg.num_layers, cfg.batch, cfg.num_kv_heads, d)).astype(np.float32))
    v = oracle.bf16_round(rng.standard_normal(k.shape).astype(np.float32))
    return q, k, v


def _run(cfg, q, k, v, **kw):
    ep = OracleEpisode(cfg, **kw)
    K, V = _prompt(cfg)
    for l in range(cfg.num_layers):
        ep.cluster_prompt(l, K, V)
    flags, outs = [], []
    for t in range(cfg.decode_steps):
        outs.append(ep.step(q[t], k[t], v[t]))
        flags.append([ep.flags[l].copy() for l in range(cfg.num_layers)])
    return ep, np.array(flags), outs


def test_flags_follow_boundaries_and_degeneracies():
    cfg = tiny_cfg()
    bset = {1, 6, 9, 15}
    q, k, v = _controlled_queries(cfg, bset)
    ep, flags, _ = _run(cfg, q, k, v)
    got = {t + 1 for t in range(cfg.decode_steps) if flags[t, 0, 0]}
    assert got == bset
    assert ep.stats["retrievals"] == len(bset)
    # S:223-224 / S:491-503: tau=1.01 -> every step; tau=-1 -> only t=1
    ep, flags, _ = _run(tiny_cfg(tau=1.01), q, k, v)
    assert flags[:, 0, 0].all() and ep.stats["retrievals"] == cfg.decode_steps
    ep, flags, _ = _run(tiny_cfg(tau=-1.0), q, k, v)
    assert flags[:, 0, 0].tolist() == [1] + [0] * (cfg.decode_steps - 1)


def test_eviction_rules_spec_examples():
    # buffer == W -> no eviction; boundary at 9 with W=8 evicts the first segment
    cfg = tiny_cfg(window_tokens=8, decode_steps=10)
    q, k, v = _controlled_queries(cfg, {1, 9})
    ep = OracleEpisode(cfg)
    K, V = _prompt(cfg)
    ep.cluster_prompt(0, K, V)
    n_prompt_units = len(ep.units(0, 0, 0))
    for t in range(8):
        ep.step(q[t], k[t], v[t])
    assert len(ep.units(0, 0, 0)) == n_prompt_units  # 8 tokens buffered == W: none evicted
    ep.step(q[8], k[8], v[8])
    units = ep.units(0, 0, 0)
    assert len(units) == n_prompt_units + 1
    P = cfg.prompt_len
    assert units[-1].positions.tolist() == list(range(P, P + 8))  # oldest segment, FIFO
    assert units[-1].uid == n_prompt_units                          # unit id = k + eviction index
    # centroid = mean of member keys, bit-exact fp32 sequential recipe
    assert np.array_equal(units[-1].centroid, oracle.segment_centroid(k[:8, 0, 0, 0]))
    # an open segment larger than W is never evicted
    cfg2 = tiny_cfg(window_tokens=4, decode_steps=9)
    q2, k2, v2 = _controlled_queries(cfg2, {1})
    ep2 = OracleEpisode(cfg2, max_open_segment=100)
    ep2.cluster_prompt(0, K, V)
    for t in range(9):
        ep2.step(q2[t], k2[t], v2[t])
    assert len(ep2.units(0, 0, 0)) == n_prompt_units
    assert len(ep2.inst[(0, 0, 0)].open_pos) == 9


def test_force_seal_and_fifo_contiguity():
    cfg = tiny_cfg(window_tokens=6, decode_steps=30)
    q, k, v = _controlled_queries(cfg, {1, 12})
    ep = OracleEpisode(cfg, max_open_segment=4)
    K, V = _prompt(cfg)
    ep.cluster_prompt(0, K, V)
    n0 = len(ep.units(0, 0, 0))
    for t in range(cfg.decode_steps):
        ep.step(q[t], k[t], v[t])
        inst = ep.inst[(0, 0, 0)]
        buffered = sum(s["pos"].size for s in inst.sealed) + len(inst.open_pos)
        assert buffered <= cfg.window_tokens or not inst.sealed
        assert len(inst.open_pos) <= 4
    segs = ep.units(0, 0, 0)[n0:]
    starts = [int(s.positions[0]) for s in segs]
    assert starts == sorted(starts)
    for s in segs:  # contiguous
        assert s.positions.tolist() == list(range(int(s.positions[0]), int(s.positions[-1]) + 1))
        assert s.positions.size <= 4


def test_coverage_every_position_exactly_once():
    cfg = tiny_cfg(decode_steps=20)
    q, k, v = _controlled_queries(cfg, {1, 4, 9, 13, 18})
    ep, _, _ = _run(cfg, q, k, v)
    inst = ep.inst[(0, 0, 0)]
    pos = list(range(inst.sinks_K.shape[0]))
    for u in inst.units:
        pos += u.positions.tolist()
    for s in inst.sealed:
        pos += s["pos"].tolist()
    pos += inst.open_pos
    assert sorted(pos) == list(range(cfg.prompt_len + cfg.decode_steps))


def test_superset_budget_equals_full_attention():
    # north_star / S:501: every unit selected => sparse attention == full attention
    cfg = tiny_cfg(budget_tokens=10_000, window_tokens=100, decode_steps=12, num_q_heads=4, num_kv_heads=2)
    rng = np.random.default_rng(3)
    q = oracle.bf16_round(rng.standard_normal((12, 1, 1, 4, 16)).astype(np.float32))
    k = oracle.bf16_round(rng.standard_normal((12, 1, 1, 2, 16)).astype(np.float32))
    v = oracle.bf16_round(rng.standard_normal((12, 1, 1, 2, 16)).astype(np.float32))
    ep = OracleEpisode(cfg)
    K, V = _prompt(cfg)
    ep.cluster_prompt(0, K, V)
    for t in range(12):
        out = ep.step(q[t], k[t], v[t])[0]
        for h in range(2):
            Kf = np.concatenate([K[0, :, h], k[:t + 1, 0, 0, h]])
            Vf = np.concatenate([V[0, :, h], v[:t + 1, 0, 0, h]])
            full = oracle.attention_f64(q[t, 0, 0, 2 * h:2 * h + 2], Kf, Vf)
            assert np.max(np.abs(out[0, 2 * h:2 * h + 2] - full)) < 1e-9
    # retrieval every step with a tiny window: the set is everything except the segment
    # evicted by THIS step's append, which follows the retrieval (R-AMB15)
    cfg2 = tiny_cfg(budget_tokens=10_000, window_tokens=3, decode_steps=12, tau=1.01)
    ep2 = OracleEpisode(cfg2)
    ep2.cluster_prompt(0, K, V)
    q2 = q[:, :, :, :2]
    k2, v2 = k[:, :, :, :1], v[:, :, :, :1]
    for t in range(12):
        n_before = len(ep2.units(0, 0, 0))
        ep2.step(q2[t], k2[t], v2[t])
        pos, _, _ = ep2.attention_rows(0, 0, 0)
        missing = set(range(cfg2.prompt_len + t + 1)) - set(pos.tolist())
        evicted_now = set()
        for u in ep2.units(0, 0, 0)[n_before:]:
            evicted_now |= set(u.positions.tolist())
        assert missing == evicted_now
        assert len(pos) == len(set(pos.tolist()))


def test_last_retrieval_reference_and_shared_mode():
    cfg = tiny_cfg(num_layers=2, decode_steps=10, tau=0.9)
    q, k, v = _controlled_queries(cfg, {1, 5})
    # drift: within a segment the query slowly rotates, so PREV_STEP never fires but
    # LAST_RETRIEVAL (anchored at the last retrieval query) eventually does.
    for t in range(10):
        q[t, :, :, :, 1] = 0.12 * (t % 4)
    ep_p, fl_p, _ = _run(cfg, q, k, v, trigger_ref=PREV_STEP)
    ep_l, fl_l, _ = _run(cfg, q, k, v, trigger_ref=LAST_RETRIEVAL)
    assert fl_l[:, 0, 0].sum() >= fl_p[:, 0, 0].sum()
    # SHARED: every layer copies the designated layer's decision
    q2 = q.copy()
    q2[:, 1] = np.roll(q2[:, 1], 3, axis=0)
    ep_s, fl_s, _ = _run(cfg, q2, k, v, boundary_mode=SHARED, shared_layer=0)
    assert np.array_equal(fl_s[:, 1], fl_s[:, 0])


def test_planted_boundary_recovery_on_generator():
    # SPEC acceptance 5: >= 95% of planted boundaries recovered by the tau rule
    cfg = synth.configs.C2.replace(num_layers=1, decode_steps=200, full_cache_layers=(),
                                   prompt_len=64, sink_tokens=0)
    q, _, _, bset = synth.decode_stream(cfg, 200, seed=0)
    q = q.float().numpy()
    fired = {1}
    for t in range(2, 201):
        if oracle.trigger_r1(q[t - 2, 0, 0], q[t - 1, 0, 0], t, cfg.tau)[0]:
            fired.add(t)
    planted = bset[0]
    assert len(fired & planted) >= 0.95 * len(planted)
    assert len(fired - planted) <= 0.05 * len(planted)


def test_offload_fetch_conservation():
    cfg = tiny_cfg(decode_steps=20, tau=1.01)
    q, k, v = _controlled_queries(cfg, {1})
    ep, _, _ = _run(cfg, q, k, v)
    inst = ep.inst[(0, 0, 0)]
    pool_rows = sum(u.positions.size for u in inst.units)
    assert ep.stats["bytes_d2h"] == pool_rows * 2 * 2 * cfg.head_dim
    # budget law: retrieved rows <= B at every step
    assert sum(inst.units[u].positions.size for u in inst.selected) <= cfg.budget_tokens



def test_fixed_stride_trigger_pattern_and_segments():
    """trigger_stride = k (P:446 fixed-stride ablation): flags exactly at t = 1, 1+k, 1+2k, ...
    whatever r_t is (the controlled queries put semantic boundaries elsewhere), and every evicted
    output segment is k tokens long (segments are sealed at the flags)."""
    cfg = tiny_cfg(decode_steps=30, window_tokens=8)
    q, k, v = _controlled_queries(cfg, {1, 7, 19})
    n_prompt_units = -(-(cfg.prompt_len - cfg.sink_tokens) // cfg.avg_cluster_size)
    for kk in (1, 3, 5):
        ep, flags, _ = _run(cfg, q, k, v, trigger_stride=kk)
        assert flags[:, 0, 0].tolist() == [1 if t % kk == 0 else 0 for t in range(cfg.decode_steps)], kk
        seg_sizes = [u.positions.size for u in ep.units(0, 0, 0)[n_prompt_units:]]
        assert seg_sizes and all(n == kk for n in seg_sizes), (kk, seg_sizes)


@pytest.mark.parametrize("n,p,sizes", [(10, 4, [4, 4, 2]), (32, 16, [16, 16]), (1, 16, [1])])
def test_page_units_spec_examples(n, p, sizes):
    """SPEC build_pages (paper §3.1 P:63 fixed-size pages, page size 16 at P:143): n
    positions in consecutive pages of p (last one short), each centroid the mean of its keys."""
    cfg = tiny_cfg(prompt_len=n + 4, sink_tokens=4, avg_cluster_size=p)
    K, V = _prompt(cfg, 3)
    ep = OracleEpisode(cfg)
    assign = np.broadcast_to((np.arange(n) // p).astype(np.int32), (1, 1, n)).copy()
    ep.cluster_prompt(0, K, V, assign=assign)
    units = ep.units(0, 0, 0)
    assert [u.positions.size for u in units] == sizes
    start = 4
    for u, sz in zip(units, sizes):
        assert u.positions.tolist() == list(range(start, start + sz))
        np.testing.assert_allclose(u.centroid, K[0, start:start + sz, 0].astype(np.float64).mean(0), rtol=0, atol=1e-6)
        start += sz
