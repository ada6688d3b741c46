"""Round-2 pins of the oracle parts the round-1 review found unpinned (VERDICT "What's weak" 1):
R1's fixed summation tree at the production head_dim, the empty-cluster repair rule (R-AMB9) and
the mode-1 (bf16 centroid operand, R-AMB10) distance. Every expected value here is either a
closed form worked by hand in the comments, or a textbook formula evaluated exactly."""
import math

import numpy as np
import pytest

import oracle


# ---------------------------------------------------------------- R1 at d = 64 / 128
def _grid_vec(rng, d):
    # multiples of 1/16 in [-8, 8): every product is a multiple of 2^-8 and |sum| < 2^13, so every
    # partial sum of dot / ||a||^2 / ||b||^2 is EXACT in fp64 whatever the summation order
    return (rng.integers(-128, 128, size=d) / 16.0).astype(np.float32)


@pytest.mark.parametrize("d", [64, 128])
def test_cosine_r1_equals_textbook_when_sums_are_exact(d):
    """P:104 cos(a, b) = a.b / (||a|| ||b||). With exactly representable partial sums the R1 tree
    order cannot matter, so R1 must equal the textbook fp64 evaluation BITWISE; a chunk bound that
    dropped or double-counted a dimension would break this."""
    rng = np.random.default_rng(d)
    for _ in range(200):
        a, b = _grid_vec(rng, d), _grid_vec(rng, d)
        A, B = a.astype(np.float64), b.astype(np.float64)
        na, nb = float(np.dot(A, A)), float(np.dot(B, B))
        ref = 0.0 if na == 0 or nb == 0 else float(np.dot(A, B)) / (math.sqrt(na) * math.sqrt(nb))
        ref = min(1.0, max(-1.0, ref))
        assert oracle.cosine_r1(a, b) == ref


@pytest.mark.parametrize("d", [64, 128])
def test_cosine_r1_every_dimension_counts(d):
    """Zeroing any single dimension of a changes R1's result, and it changes it to exactly the
    textbook cosine of the modified vector (so no dimension is dropped or counted twice)."""
    rng = np.random.default_rng(100 + d)
    a = _grid_vec(rng, d)
    a[a == 0] = 0.5
    b = _grid_vec(rng, d)
    b[b == 0] = -0.25
    base = oracle.cosine_r1(a, b)
    for e in range(d):
        a2 = a.copy()
        a2[e] = 0.0
        A, B = a2.astype(np.float64), b.astype(np.float64)
        ref = float(np.dot(A, B)) / (math.sqrt(float(np.dot(A, A))) * math.sqrt(float(np.dot(B, B))))
        got = oracle.cosine_r1(a2, b)
        assert got != base and got == ref, e


@pytest.mark.parametrize("d", [64, 128])
def test_cosine_r1_random_normal_within_fp64_rounding(d):
    """On general fp32 inputs R1 differs from the textbook fp64 formula only by summation-order
    rounding: |delta| <= (d + 4) eps64 * sum|a_e b_e| / (||a|| ||b||) + 8 eps64 (standard bound)."""
    rng = np.random.default_rng(7 + d)
    eps = np.finfo(np.float64).eps
    for _ in range(300):
        a = rng.standard_normal(d).astype(np.float32)
        b = (0.3 * a + rng.standard_normal(d)).astype(np.float32)
        A, B = a.astype(np.float64), b.astype(np.float64)
        nA, nB = math.sqrt(float(np.dot(A, A))), math.sqrt(float(np.dot(B, B)))
        ref = float(np.dot(A, B)) / (nA * nB)
        bound = (d + 4) * eps * float(np.abs(A * B).sum()) / (nA * nB) + 8 * eps
        got = oracle.cosine_r1(a, b)
        assert abs(got - ref) <= bound, (got, ref, bound)
        assert abs(got - ref) <= 1e-15 * max(1.0, abs(ref)) * (d / 16)  # ~1e-15 relative scale


def test_trigger_r1_d128_mean_of_head_cosines():
    """r_t = (1/H) sum_h cos(q_ref^h, q_t^h) at H = 32, d = 128: head h is parallel
    (cos 1), anti-parallel (cos -1) or orthogonal (cos 0) by h % 4, so r is a
    hand-computable rational (16 parallel, 8 anti-parallel, 8 orthogonal -> r = 8/32 = 0.25)."""
    H, d = 32, 128
    rng = np.random.default_rng(3)
    q_ref = np.zeros((H, d), np.float32)
    q_cur = np.zeros((H, d), np.float32)
    want = 0.0
    for h in range(H):
        v = _grid_vec(rng, d)
        v[0] = 1.0
        q_ref[h] = v
        kind = h % 4
        if kind in (0, 3):      # parallel (scaled by 2): cos = 1
            q_cur[h] = 2 * v
            want += 1.0
        elif kind == 1:    # anti-parallel: cos = -1
            q_cur[h] = -v
            want -= 1.0
        else:              # orthogonal: a vector supported where v is zero, else swap trick
            w = np.zeros(d, np.float32)
            w[1], w[2] = v[2], -v[1]   # v.w = v1 v2 - v2 v1 = 0 exactly
            if w[1] == 0 and w[2] == 0:
                w[3], w[4] = v[4], -v[3]
            q_cur[h] = w
    want /= H
    assert want == 0.25
    flag, r = oracle.trigger_r1(q_ref, q_cur, 5, want - 1e-12)
    # (each +-1 cosine carries at most a few ulp from the two square roots)
    assert abs(r - want) <= 4 * H * np.finfo(np.float64).eps / H and flag == 0
    flag, r = oracle.trigger_r1(q_ref, q_cur, 5, want + 1e-12)
    assert flag == 1
    # a head-count slip (dividing by H - 1, or skipping a head) moves r by >= 1/32


# ---------------------------------------------------------------- repair (R-AMB9), hand-worked
def test_kmeans_repair_hand_worked_example():
    """d = 1, X = [12, 12, 17, 11, 5, 11, 5], k = 4, 2 iterations (exact mode), worked by hand:

    init (R-AMB8, x_{floor(jN/k)}, N=7): indices 0, 1, 3, 5 -> C = [12, 12, 11, 11]
    iter 1 assign (ties -> lower j): x0,x1 -> 0 (d 0); x2=17 -> 0 (25 < 36); x3 -> 2 (0);
      x4=5 -> 2 (36 < 49); x5 -> 2 (0); x6=5 -> 2 (36). counts [3,0,4,0], E = [1, 3]
    repair E[0]=1: largest dmin among clusters with >= 2 members: x4 and x6 tie at 36 -> lower
      index x4 -> cluster 1. counts [3,1,3,0]
    repair E[1]=3: x6 (36) -> cluster 3. counts [3,1,2,1]
    update: C = [41/3, 5, 11, 5]
    iter 2 assign: x0,x1=12 -> 2 (1 < (5/3)^2); x2=17 -> 0 ((10/3)^2 = 11.1); x3,x5 -> 2 (0);
      x4,x6=5 -> 1 (tie with 3 at 0 -> lower). counts [1,2,4,0], E = [3]
    repair E[0]=3: x2 has the largest dmin (11.1) but its cluster 0 is a singleton -> not
      eligible; eligible maximum 1 at x0 and x1 -> lower index x0 -> cluster 3
    update: C = [17, 5, 34/3, 12]; final assign [3, 2, 0, 2, 1, 2, 1]

    A "smallest dmin" rule, a rule ignoring the >= 2-member condition, or ties -> higher index
    each give a different result."""
    X = np.array([[12], [12], [17], [11], [5], [11], [5]], np.float32)
    a, C, counts, J, dmin = oracle.kmeans(X, 4, 2, mode=0)
    assert a.tolist() == [3, 2, 0, 2, 1, 2, 1]
    assert counts.tolist() == [1, 2, 3, 1]
    assert np.array_equal(C[:, 0], np.array([17, 5, 34 / 3, 12], np.float32))
    # after one iteration (the first repair only)
    a1, C1, counts1, _, dmin1 = oracle.kmeans(X, 4, 1, mode=0)
    assert a1.tolist() == [0, 0, 0, 2, 1, 2, 3]
    assert np.array_equal(C1[:, 0], np.array([41 / 3, 5, 11, 5], np.float32))
    assert dmin1.tolist() == [0, 0, 25, 0, 0, 0, 0]  # donors' dmin reset to 0
    # mode 1 (bf16 centroid operand) reaches the same decisions on this input
    a_m1 = oracle.kmeans(X, 4, 2, mode=1)[0]
    assert a_m1.tolist() == [3, 2, 0, 2, 1, 2, 1]


# ---------------------------------------------------------------- mode-1 distance (R-AMB10)
def test_kmeans_mode1_distance_closed_form():
    """Mode 1 evaluates ||x||^2 - 2 x.bf16(c) + ||c||^2 with ||c||^2 of the fp32 centroid.
    X = [[1, 0], [1 + 2^-7, 0]], k = 1, 2 iterations: after iteration 1, c = (1 + 2^-8, 0), which
    is not a bf16 value; bf16(c) = (1, 0) (RNE tie -> even). Iteration 2 dmin of x0 = [1, 0]:
      1 - 2*1*1 + (1 + 2^-8)^2 = 2^-7 + 2^-16 = 0.0078277587890625   (exact in fp64)
    and of x1: (1+2^-7)^2 - 2(1+2^-7) + (1+2^-8)^2 = 2^-14 - 2^-7... worked: (1+a)^2 - 2(1+a) +
    (1+b)^2 with a = 2^-7, b = 2^-8 -> a^2 - 1 + 1 + 2b + b^2 = 2^-14 + 2^-7 + 2^-16.
    Exact mode gives (2^-8)^2 = 2^-16 for both; using ||bf16(c)||^2 instead would give 0 for x0."""
    X = np.array([[1.0, 0.0], [1.0 + 2 ** -7, 0.0]], np.float32)
    _, C, _, _, dmin = oracle.kmeans(X, 1, 2, mode=1)
    assert C[0, 0] == np.float32(1 + 2 ** -8)
    assert dmin[0] == np.float32(2 ** -7 + 2 ** -16)
    assert dmin[1] == np.float32(2 ** -14 + 2 ** -7 + 2 ** -16)
    _, _, _, _, dmin0 = oracle.kmeans(X, 1, 2, mode=0)
    assert dmin0.tolist() == [2 ** -16, 2 ** -16]


def test_kmeans_mode1_within_bf16_operand_bound_of_exact():
    """|dist_mode1 - dist_exact| = |2 x.(c - bf16(c))| <= 2 ||x|| ||c - bf16(c)|| (Cauchy-Schwarz),
    plus fp64 rounding. The final dmin of every key (mode 1) is checked against the exact squared
    distance to its assigned fp32 centroid under that bound; on bf16-exact centroids (iteration 1:
    the init centroids are keys) the two modes agree to fp64 rounding."""
    rng = np.random.default_rng(11)
    X = oracle.bf16_round((rng.standard_normal((400, 128)) + np.repeat(rng.standard_normal((20, 128)) * 2, 20, 0))
                          .astype(np.float32))
    k = 25
    # iteration 1 only: the centroids used by the assignment are keys (bf16 exact)
    a1, _, _, _, dm1 = oracle.kmeans(X, k, 1, mode=1)
    N = len(X)
    C0 = np.stack([X[(j * N) // k] for j in range(k)]).astype(np.float64)
    Xd = X.astype(np.float64)
    D0 = ((Xd[:, None, :] - C0[None]) ** 2).sum(-1)
    assert np.array_equal(a1, np.argmin(D0, axis=1))   # no empty cluster on this input
    assert np.allclose(dm1, D0.min(1), rtol=1e-6, atol=1e-6)  # (dmin is returned as fp32)
    # several iterations: centroids are fp32 means (not bf16); final dmin vs the exact distance
    # to the centroids the last assignment used (the previous update) is within the operand bound
    a5, C5, _, _, dm5 = oracle.kmeans(X, k, 5, mode=1)
    _, C4, _, _, _ = oracle.kmeans(X, k, 4, mode=1)
    C4d = C4.astype(np.float64)
    Cb = oracle.bf16_round(C4).astype(np.float64)
    exact = ((Xd - C4d[a5]) ** 2).sum(-1)
    bound = 2 * np.linalg.norm(Xd, axis=1) * np.linalg.norm(C4d[a5] - Cb[a5], axis=1) + 1e-9 * (1 + exact)
    assert np.all(np.abs(dm5.astype(np.float64) - exact) <= bound + 1e-6 * (1 + exact))
    # and the assignment is the argmin of the mode-1 expression over ALL centroids
    D1 = (Xd ** 2).sum(1)[:, None] - 2 * Xd @ Cb.T + (C4d ** 2).sum(1)[None]
    assert np.array_equal(a5, np.argmin(D1, axis=1))
