"""GPU k-means (louiskv_cluster_prompt, tcgen05 assignment) vs the oracle at the sizes the real
configs use ("employs the k-means clustering algorithm ... calculates the centroid"):

* C2 size (N = 32736 keys, k = 2046 centroids = 8 N-tiles of 256) with one Lloyd iteration from the
  shared strided init (R-AMB8), so both sides assign against the very same centroids: every key's
  cluster must equal the oracle's, except keys whose two candidate distances are within the
  fp32-accumulation bound of the bf16-operand contraction (each such key checked individually);
* a repair-forcing input (k = 512 > 256, 256 empty clusters after the first assignment, ties across
  N-tiles) whose units (sizes, members, centroids) must equal the oracle's after 1-3 iterations;
* the overlapping C1 input at one iteration, mismatches checked key by key (near ties only).
"""
import concurrent.futures as cf

import numpy as np
import pytest
import torch

import oracle
from synth.configs import C1, C2

from _pair import make_inputs, np32

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def _lkv():
    import paper_2510_11292_b200 as lkv
    return lkv


def gpu_assign(ctx, l, b, h, N, S):
    """Per-key unit id of the GPU clustering (from the cluster-major pool order) + fp32 centroids."""
    cen, sizes, first = ctx.get_units(l, b, h)
    pos = ctx.get_unit_positions(l, b, h)
    a = np.full(N, -1, np.int32)
    o = 0
    for j, s in enumerate(sizes):
        a[pos[o:o + s] - S] = j
        o += s
    assert (a >= 0).all()
    return a, cen, sizes


def near_tie_check(X, C_used, a_g, a_o, d=128):
    """Every key the GPU assigns differently from the oracle (mode 1, R-AMB10) must be a near tie:
    with s_j = x.bf16(c_j) - ||c_j||^2/2, the GPU (fp32 accumulation of exact bf16 products, fp32
    half-norm) errs by at most gamma (sum_e |x_e bf16(c_je)| + ||c_j||^2/2), gamma = (d+4) 2^-24, so
    the exact mode-1 distances of the two candidates differ by at most 2 (err_jg + err_jo).
    Returns (n_mismatch, worst gap / bound)."""
    mis = np.nonzero(a_g != a_o)[0]
    if mis.size == 0:
        return 0, 0.0
    Xd = X[mis].astype(np.float64)
    Cd = C_used.astype(np.float64)
    Cb = oracle.bf16_round(C_used).astype(np.float64)
    gam = (d + 4) * U32
    worst = 0.0
    for t, i in enumerate(mis):
        x = Xd[t]
        jg, jo = int(a_g[i]), int(a_o[i])
        dist = lambda j: float(x @ x - 2 * x @ Cb[j] + Cd[j] @ Cd[j])
        err = lambda j: gam * (float(np.abs(x * Cb[j]).sum()) + 0.5 * float(Cd[j] @ Cd[j]))
        gap = dist(jg) - dist(jo)
        bound = 2 * (err(jg) + err(jo))
        assert gap >= -1e-9 * (1 + abs(dist(jo))), (i, jg, jo, gap)  # the oracle's choice is optimal
        assert gap <= bound, (i, jg, jo, gap, bound)
        worst = max(worst, gap / bound)
    return int(mis.size), worst


@pytest.mark.timeout(1800)
def test_kmeans_c2_size_one_iteration_vs_oracle():
    """C2 geometry (32K prompt, S = 32, c = 16 -> k = 2046, 8 tcgen05 N-tiles), overlapping planted
    data (k/4 planted groups scattered over positions, the throughput recipe), 2 KV heads, ONE Lloyd
    iteration: both sides assign against the strided init centroids (keys, bf16 exact)."""
    lkv = _lkv()
    cfg = C2.replace(num_layers=1, full_cache_layers=(), num_kv_heads=2, num_q_heads=8, kmeans_iters=1,
                     k_planted=2046 // 4)
    inp = make_inputs(cfg, 1, 21)
    ctx = lkv.Context(lkv.make_config(cfg))
    ctx.cluster_prompt(0, inp.K[0], inp.V[0])
    assert ctx.stats()["kmeans_tc_iters"] == 1
    S, N, k = 32, 32736, 2046
    Xall = np32(inp.K[0])[0]

    def oracle_head(h):
        return oracle.kmeans(Xall[S:, h].copy(), k, 1, mode=1)

    with cf.ThreadPoolExecutor(2) as ex:  # (ctypes releases the GIL)
        res = list(ex.map(oracle_head, range(2)))
    tot_mis = 0
    for h in range(2):
        X = Xall[S:, h]
        a_o, C_o, cnt_o, _, _ = res[h]
        a_g, C_g, sizes = gpu_assign(ctx, 0, 0, h, N, S)
        assert (np.bincount(a_g, minlength=k) >= 1).all() and (cnt_o >= 1).all()
        C_init = np.stack([X[(j * N) // k] for j in range(k)])
        n_mis, worst = near_tie_check(X, C_init, a_g, a_o)
        tot_mis += n_mis
        print(f"head {h}: {n_mis} of {N} keys assigned differently (all near ties, worst gap/bound "
              f"{worst:.3f})")
        assert n_mis <= N // 1000
        # centroids of the GPU clustering = means of its members (1e-3 relative, fp32)
        C_ref = oracle.centroids_of(X, a_g, k).astype(np.float64)
        scale = np.maximum(np.abs(C_ref), 1e-3 * np.abs(C_ref).max())
        assert (np.abs(C_g - C_ref) / scale).max() < 1e-3
        # where the memberships agree the centroids agree with the oracle's
        same = np.ones(k, bool)
        same[np.unique(np.concatenate([a_g[a_g != a_o], a_o[a_g != a_o]]))] = False
        assert (np.abs(C_g[same] - C_o[same]) / scale[same]).max() < 1e-3
        # every column block of 256 centroids (each tcgen05 N-tile) really receives its own keys
        per_tile = np.bincount(a_g // 256, minlength=8)
        assert (per_tile > 0).all() and per_tile.sum() == N
    ctx.close()


def _repair_input(n_heads=2, seed=0):
    """Keys of one layer [1, P, H, d] (S = 0, N = 8192, c = 16 -> k = 512): block B = p // 16 holds
    mu_{B mod 256} (mu_m = +-8 e_{m mod 128}), so the strided init (position 16 j) seeds centroid j and
    j + 256 with the SAME key: every tie goes to the lower id (across tcgen05 N-tiles 0 and 1) and
    clusters 256..511 are empty after the first assignment (E = 256). One outlier per block (offset
    1 + B % 15, never an init position) is mu_m + delta e_{(m+1) mod 128}, the 512 deltas a random
    permutation of the 512 bf16 values in [0.5, 8): squared distances delta^2 are distinct with gaps
    >= 2^-8, far above fp32 rounding, so the repair's donor order (largest dmin first, R-AMB9) is
    unambiguous."""
    d, N = 128, 8192
    rng = np.random.default_rng(seed)
    deltas = np.concatenate([0.5 + np.arange(128) / 256, 1 + np.arange(128) / 128, 2 + np.arange(128) / 64,
                             4 + np.arange(128) / 32]).astype(np.float32)
    K = np.zeros((1, N, n_heads, d), np.float32)
    for h in range(n_heads):
        perm = rng.permutation(512)
        for B in range(512):
            m = B % 256
            mu = np.zeros(d, np.float32)
            mu[m % 128] = 8.0 if m < 128 else -8.0
            K[0, 16 * B:16 * B + 16, h] = mu
            o = 16 * B + 1 + B % 15
            K[0, o, h] = mu
            K[0, o, h, (m + 1) % 128] += deltas[perm[B]]
    assert np.array_equal(oracle.bf16_round(K), K)
    V = rng.standard_normal(K.shape).astype(np.float32)
    return K, oracle.bf16_round(V)


@pytest.mark.parametrize("iters", [1, 2, 3])
def test_kmeans_repair_forcing_units_equal_oracle(iters):
    lkv = _lkv()
    H = 2
    cfg = C1.replace(num_kv_heads=H, num_q_heads=H, prompt_len=8192, sink_tokens=0, avg_cluster_size=16,
                     clusters_override=0, kmeans_iters=iters)
    K, V = _repair_input(H)
    Kd = torch.from_numpy(K).to("cuda", torch.bfloat16)
    Vd = torch.from_numpy(V).to("cuda", torch.bfloat16)
    ctx = lkv.Context(lkv.make_config(cfg))
    ctx.cluster_prompt(0, Kd, Vd)
    assert ctx.stats()["kmeans_tc_iters"] == iters
    for h in range(H):
        X = K[0, :, h]
        a_o, C_o, cnt_o, _, dmin_o = oracle.kmeans(X, 512, iters, mode=1)
        if iters == 1:
            # the design: 256 empty clusters filled by the 256 largest-delta outliers, in dmin order
            assert (cnt_o[256:] == 1).all()
        a_g, C_g, sizes = gpu_assign(ctx, 0, 0, h, 8192, 0)
        assert np.array_equal(a_g, a_o), (h, np.nonzero(a_g != a_o)[0][:10])
        assert np.array_equal(sizes, cnt_o)
        scale = np.maximum(np.abs(C_o), 1e-3 * np.abs(C_o).max())
        assert (np.abs(C_g - C_o) / scale).max() < 1e-3
    ctx.close()


@pytest.mark.parametrize("impl", [0, 1])
def test_kmeans_overlapping_one_iteration_near_ties_checked(impl):
    """C1 (N = 4096, k = 64), 16 planted groups scattered over positions (so several init centroids
    share a group and keys sit between them): one iteration, each mismatched key a proven near tie."""
    lkv = _lkv()
    cfg = C1.replace(k_planted=16, kmeans_iters=1, num_kv_heads=1)
    inp = make_inputs(cfg, 1, 1)
    ctx = lkv.Context(lkv.make_config(cfg, kmeans_impl=impl))
    ctx.cluster_prompt(0, inp.K[0], inp.V[0])
    X = np32(inp.K[0])[0, :, 0]
    a_o = oracle.kmeans(X, 64, 1, mode=1)[0]
    a_g, C_g, _ = gpu_assign(ctx, 0, 0, 0, 4096, 0)
    C_init = np.stack([X[(j * 4096) // 64] for j in range(64)])
    n_mis, worst = near_tie_check(X, C_init, a_g, a_o)
    print(f"impl {impl}: {n_mis} mismatches, worst gap/bound {worst:.3f}")
    assert n_mis <= 8
    ctx.close()
