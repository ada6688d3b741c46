"""Pins for the oracle's selection, k-means, centroid and attention."""
import itertools
import math

import numpy as np
import pytest

import oracle


# ---------------------------------------------------------------- selection
def test_select_spec_examples():
    # S:349-351
    assert oracle.select_greedy([.9, .8, .5], [3, 2, 2], 5).tolist() == [0, 1]
    assert oracle.select_greedy([.9, .8, .5], [3, 2, 2], 0).tolist() == []
    assert oracle.select_greedy([.9, .8], [10, 2], 4).tolist() == [1]
    # survey counterexample to whole-set monotonicity: {0,2} at B=4, {0,1} at B=5
    assert oracle.select_greedy([.9, .8, .7], [3, 2, 1], 4).tolist() == [0, 2]
    assert oracle.select_greedy([.9, .8, .7], [3, 2, 1], 5).tolist() == [0, 1]


def _greedy_characterization_holds(A, sizes, B, sel):
    """Specification of skip-and-continue greedy, checked without running it:
    rank = (A desc, id asc); a unit is in S iff it fits the budget left by the
    members of S ranked before it."""
    order = sorted(range(len(A)), key=lambda u: (-float(A[u]), u))
    S = set(sel)
    used = 0
    for u in order:
        fits = used + sizes[u] <= B
        if (u in S) != fits:
            return False
        if fits:
            used += sizes[u]
    return used <= B


def test_select_matches_specification_random_and_brute_force():
    rng = np.random.default_rng(0)
    for trial in range(500):
        n = int(rng.integers(1, 13))
        A = rng.random(n).astype(np.float32)
        if trial % 3 == 0:  # exact ties -> lower id first
            A[rng.integers(0, n, size=n // 2)] = A[0]
        sizes = rng.integers(1, 9, size=n).astype(np.int32)
        B = int(rng.integers(0, 40))
        sel = oracle.select_greedy(A, sizes, B)
        assert sizes[sel].sum() <= B
        assert list(sel) == sorted(sel)
        assert _greedy_characterization_holds(A, sizes, B, sel)
        # brute force: among all feasible subsets, greedy's set is the unique one
        # satisfying the characterization (enumerate all 2^n subsets)
        n_ok = 0
        for mask in range(1 << n):
            cand = [u for u in range(n) if mask >> u & 1]
            if _greedy_characterization_holds(A, sizes, B, cand):
                n_ok += 1
                assert cand == list(sel)
        assert n_ok == 1


def test_select_unit_sizes_equal_top_b_argsort():
    rng = np.random.default_rng(1)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        A = rng.random(n).astype(np.float32)
        A[rng.integers(0, n, size=n // 3)] = A[0]
        B = int(rng.integers(0, n + 5))
        sel = oracle.select_greedy(A, np.ones(n, np.int32), B)
        ref = np.sort(np.argsort(-A.astype(np.float64), kind="stable")[:B])
        assert np.array_equal(sel, ref)


def test_select_prefix_before_first_skip_grows_with_budget():
    rng = np.random.default_rng(2)
    for _ in range(200):
        n = int(rng.integers(1, 30))
        A = rng.random(n).astype(np.float32)
        sizes = rng.integers(1, 10, size=n).astype(np.int32)
        order = sorted(range(n), key=lambda u: (-float(A[u]), u))

        def prefix(B):
            sel = set(oracle.select_greedy(A, sizes, B).tolist())
            p = []
            for u in order:
                if u not in sel:
                    break
                p.append(u)
            return p

        prev = []
        for B in range(0, 60, 3):
            p = prefix(B)
            assert p[:len(prev)] == prev
            prev = p


# ---------------------------------------------------------------- k-means
def _blobs(rng, k, per, d, sep=10.0, noise=0.3, shuffle=True):
    """Blob-major layout (blob j at rows [j*per, (j+1)*per)) so the strided
    init x_{floor(jN/k)} seeds one centroid per blob; with shuffle=False
    rows are shuffled (and the seeding guarantee is lost)."""
    centers = rng.standard_normal((k, d)) * sep
    X = np.concatenate([centers[j] + noise * rng.standard_normal((per, d)) for j in range(k)])
    lab = np.repeat(np.arange(k), per)
    if shuffle:
        perm = rng.permutation(len(X))
        return oracle.bf16_round(X[perm].astype(np.float32)), lab[perm]
    return oracle.bf16_round(X.astype(np.float32)), lab


def test_kmeans_k1_is_global_mean():
    rng = np.random.default_rng(0)
    X = oracle.bf16_round(rng.standard_normal((200, 16)).astype(np.float32))
    a, C, counts, J, _ = oracle.kmeans(X, 1, 3, mode=0)
    assert (a == 0).all() and counts[0] == 200
    assert np.allclose(C[0], X.astype(np.float64).mean(0), rtol=0, atol=1e-6)


def test_kmeans_spec_two_groups_recovered():
    # 20 points near [10,0] and 20 near [-10,0]
    rng = np.random.default_rng(1)
    X = np.concatenate([np.array([10, 0]) + 0.5 * rng.standard_normal((20, 2)),
                        np.array([-10, 0]) + 0.5 * rng.standard_normal((20, 2))]).astype(np.float32)
    a, C, counts, J, _ = oracle.kmeans(X, 2, 10, mode=0)
    assert len(set(a[:20])) == 1 and len(set(a[20:])) == 1 and a[0] != a[20]


def test_kmeans_identical_keys_repair():
    # all keys identical, k=2 -> two non-empty clusters
    X = np.ones((10, 4), np.float32)
    a, C, counts, J, _ = oracle.kmeans(X, 2, 5, mode=1)
    assert counts.min() >= 1 and counts.sum() == 10
    # retrievable 17, c=16 -> k=2, both non-empty
    X = oracle.bf16_round(np.random.default_rng(2).standard_normal((17, 8)).astype(np.float32))
    a, C, counts, J, _ = oracle.kmeans(X, math.ceil(17 / 16), 10, mode=1)
    assert (counts >= 1).all() and counts.sum() == 17


@pytest.mark.parametrize("mode", [0, 1])
def test_kmeans_planted_recovery_partition_fixed_point(mode):
    rng = np.random.default_rng(3)
    X, lab = _blobs(rng, 12, 30, 32, shuffle=False)
    a, C, counts, J, _ = oracle.kmeans(X, 12, 10, mode=mode)
    # partition: every key in exactly one cluster, no empties
    assert counts.sum() == len(X) and (counts >= 1).all()
    assert np.array_equal(np.bincount(a, minlength=12), counts)
    # fixed point: stored centroid = mean of members
    for j in range(12):
        m = X[a == j].astype(np.float64).mean(0)
        assert np.allclose(C[j], m, rtol=1e-6, atol=1e-6)
    # planted groups recovered exactly (up to relabelling)
    pairs = set(zip(a.tolist(), lab.tolist()))
    assert len(pairs) == 12


def test_kmeans_objective_non_increasing_exact_mode():
    rng = np.random.default_rng(4)
    X = oracle.bf16_round((rng.standard_normal((600, 16)) + np.repeat(rng.standard_normal((30, 16)) * 0.8, 20, 0)).astype(np.float32))
    a, C, counts, J, _ = oracle.kmeans(X, 40, 15, mode=0)
    assert np.all(np.diff(J) <= 1e-9 * J[0])
    assert (counts >= 1).all()


def test_kmeans_matches_sklearn_lloyd():
    from sklearn.cluster import KMeans
    rng = np.random.default_rng(5)
    X, _ = _blobs(rng, 8, 25, 16, sep=3.0, noise=1.0)
    k, iters = 8, 6
    a, C, counts, J, _ = oracle.kmeans(X, k, iters, mode=0)
    N = len(X)
    C0 = np.stack([X[(j * N) // k] for j in range(k)]).astype(np.float64)
    km = KMeans(n_clusters=k, init=C0, n_init=1, algorithm="lloyd", tol=0.0, max_iter=iters).fit(X.astype(np.float64))
    assert (counts >= 1).all()
    assert np.allclose(km.cluster_centers_, C.astype(np.float64), rtol=0, atol=1e-5)


def test_kmeans_tiny_converged_is_lloyd_fixed_point():
    rng = np.random.default_rng(6)
    X = oracle.bf16_round(rng.standard_normal((10, 3)).astype(np.float32))
    a, C, counts, J, _ = oracle.kmeans(X, 3, 60, mode=0)
    D = ((X[:, None, :].astype(np.float64) - C[None].astype(np.float64)) ** 2).sum(-1)
    assert np.array_equal(a, np.argmin(D, axis=1))


def test_segment_centroid_closed_form():
    # S:152-154
    assert np.array_equal(oracle.segment_centroid([[1, 1]]), np.array([1, 1], np.float32))
    assert np.array_equal(oracle.segment_centroid([[0, 0], [2, 2]]), np.array([1, 1], np.float32))
    c = oracle.segment_centroid([[1, 0], [0, 1], [1, 1]])
    assert np.allclose(c, [2 / 3, 2 / 3], atol=1e-6)


def test_bf16_round_rne():
    # 1 + 2^-8 is the midpoint between 1 and 1+2^-7: ties to even -> 1
    assert oracle.bf16_round(np.array([1 + 2 ** -8], np.float32))[0] == 1.0
    assert oracle.bf16_round(np.array([1 + 3 * 2 ** -8], np.float32))[0] == 1 + 2 ** -6
    import torch
    x = np.random.default_rng(0).standard_normal(10000).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(oracle.bf16_round(x), ref)


# ---------------------------------------------------------------- attention
def test_attention_spec_closed_forms():
    # S:402-414
    o = oracle.attention_f64([[0.3, -1.0]], [[1.0, 2.0]], [[5.0, -7.0]])
    assert np.array_equal(o[0], [5.0, -7.0])
    V = np.array([[1, 2], [3, 4], [5, 9]], np.float32)
    o = oracle.attention_f64([[0, 0]], np.random.default_rng(0).standard_normal((3, 2)), V)
    assert np.allclose(o[0], V.mean(0), atol=1e-12)
    o = oracle.attention_f64([[math.log(3)]], [[1], [0]], [[1], [0]])
    assert abs(o[0, 0] - 0.75) < 1e-7  # q = fl32(ln 3): input rounding ~4e-9
    o = oracle.attention_f64([[1.0]], [[2], [1]], [[1], [0]])
    assert abs(o[0, 0] - math.e ** 2 / (math.e ** 2 + math.e)) < 1e-9
    assert abs(o[0, 0] - 0.7311) < 1e-4


def test_attention_matches_torch_sdpa():
    import torch
    rng = np.random.default_rng(7)
    q = rng.standard_normal((4, 128)).astype(np.float32)
    K = rng.standard_normal((300, 128)).astype(np.float32)
    V = rng.standard_normal((300, 128)).astype(np.float32)
    o = oracle.attention_f64(q, K, V)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q.astype(np.float64))[None], torch.from_numpy(K.astype(np.float64))[None],
        torch.from_numpy(V.astype(np.float64))[None])[0].numpy()
    assert np.allclose(o, ref, atol=1e-12)
