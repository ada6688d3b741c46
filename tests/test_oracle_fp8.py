"""Pins of the oracle's E4M3 rounding (reading R-FP8: the FP8 host-pool variant).

The oracle writes the rounding out from the format's definition (lko_e4m3_round); these pins tie it
to things other than itself: every finite bf16 value against PyTorch's float8_e4m3fn cast (an
independent library routine, round-to-nearest-even), hand-worked ties, subnormals and saturation."""
import numpy as np
import torch

import oracle


def _all_bf16_values():
    bits = np.arange(1 << 16, dtype=np.uint32) << 16
    x = bits.view(np.float32)
    return x[np.isfinite(x)]


def test_e4m3_equals_torch_cast_on_every_bf16_value():
    x = _all_bf16_values()
    x = x[np.abs(x) < 464.0]  # (torch's cast is non-saturating: 464 and above become NaN there)
    ours = oracle.e4m3_round(x)
    ref = torch.from_numpy(x.copy()).to(torch.float8_e4m3fn).to(torch.float32).numpy()
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))


def test_e4m3_hand_worked_values():
    cases = {
        1.0: 1.0, 1.0625: 1.0,          # 1 + 2^-4 is the midpoint of 1 and 1.125: tie to even (1.0)
        1.1875: 1.25,                   # 1 + 3/16: midpoint of 1.125 and 1.25, even mantissa is 1.25
        1.125: 1.125, 0.0: 0.0,
        2.0 ** -9: 2.0 ** -9,           # smallest subnormal
        2.0 ** -10: 0.0,                # half of it: tie to even (0)
        3 * 2.0 ** -11: 2.0 ** -9,      # 0.75 of the smallest subnormal rounds up
        2.0 ** -6: 2.0 ** -6,           # smallest normal
        7 * 2.0 ** -9: 7 * 2.0 ** -9,   # largest subnormal
        240.0: 240.0, 248.0: 256.0,     # binade [128, 256) has quantum 16; 248 ties to even -> 256
        448.0: 448.0, 460.0: 448.0, 500.0: 448.0, 1e30: 448.0,   # saturation (satfinite)
        -1.1875: -1.25, -1000.0: -448.0,
    }
    x = np.array(list(cases), np.float32)
    assert np.array_equal(oracle.e4m3_round(x), np.array(list(cases.values()), np.float32))


def test_e4m3_properties():
    x = _all_bf16_values()
    y = oracle.e4m3_round(x)
    assert np.array_equal(oracle.e4m3_round(y), y)                      # idempotent
    order = np.argsort(x, kind="stable")
    assert np.all(np.diff(y[order]) >= 0)                               # monotone
    assert np.array_equal(oracle.e4m3_round(-x), -y)                    # odd
    assert len(np.unique(np.abs(y))) == 1 + 7 + 15 * 8 - 1              # 0, 7 subnormals, 15 binades x 8 minus NaN
    small = np.abs(x) < 448
    rel = np.abs(y[small] - x[small]) / np.maximum(np.abs(x[small]), 2.0 ** -6)
    assert rel.max() <= 2.0 ** -4 + 1e-12                               # half a quantum of 3 mantissa bits


def test_fp8_pool_episode_changes_only_retrieved_rows():
    """With the FP8 pool, the oracle episode makes the same decisions (flags, selections, unit tables:
    centroids come from the bf16 keys), moves half the pool bytes, holds E4M3 values exactly in the
    retrieved rows, and its attention stays within the E4M3 error of the bf16-pool episode."""
    from oracle.episode import OracleEpisode
    from test_oracle_episode import tiny_cfg, _prompt, _controlled_queries
    cfg = tiny_cfg(decode_steps=30, window_tokens=6)
    q, k, v = _controlled_queries(cfg, {5, 9, 14, 20, 26})
    K, V = _prompt(cfg)
    eps = [OracleEpisode(cfg), OracleEpisode(cfg, pool_fp8=True)]
    outs = [[], []]
    for i, ep in enumerate(eps):
        ep.cluster_prompt(0, K, V)
        for t in range(cfg.decode_steps):
            outs[i].append(ep.step(q[t], k[t], v[t]))
    a, b = eps
    for key in ("retrievals", "units_scored", "units_selected", "units_reused", "units_fetched",
                "segments_evicted"):
        assert a.stats[key] == b.stats[key], key
    assert b.stats["bytes_h2d"] * 2 == a.stats["bytes_h2d"] > 0
    assert b.stats["bytes_d2h"] * 2 == a.stats["bytes_d2h"] > 0
    assert a.selection(0, 0, 0) == b.selection(0, 0, 0)
    for ua, ub in zip(a.units(0, 0, 0), b.units(0, 0, 0)):
        assert np.array_equal(ua.centroid, ub.centroid) and np.array_equal(ua.positions, ub.positions)
        assert np.array_equal(ub.K, oracle.e4m3_round(ua.K)) and np.array_equal(ub.V, oracle.e4m3_round(ua.V))
    err = max(np.abs(x - y).max() for x, y in zip(outs[0], outs[1]))
    assert 0 < err < 2.0 ** -4 * 4  # rows within 2^-4 relative, |v| ~ N(0,1)
