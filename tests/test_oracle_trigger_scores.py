"""Pins for the oracle's trigger (R1), exp (R3) and group scores (R2).

Each check is fixed by the paper / SPEC closed forms or by an invariant of the
mathematics, never by re-typing the oracle's own formula.
"""
import math

import numpy as np
import pytest

import oracle


# ---------------------------------------------------------------- cosine / r_t
def test_cosine_spec_examples():
    # S:38-40
    assert oracle.cosine_r1([1, 0], [1, 0]) == 1.0
    assert oracle.cosine_r1([1, 0], [0, 1]) == 0.0
    assert abs(oracle.cosine_r1([1, 1], [1, 0]) - 0.70710678) < 1e-6
    # Pythagorean closed form: [3,4]·[4,3] / 25 = 24/25 exactly representable steps
    assert abs(oracle.cosine_r1([3, 4], [4, 3]) - 0.96) < 1e-15
    # zero norm -> 0
    assert oracle.cosine_r1([0, 0], [1, 2]) == 0.0


def test_cosine_symmetry_and_power_of_two_scale_invariance():
    rng = np.random.default_rng(0)
    for _ in range(50):
        a = rng.standard_normal(128).astype(np.float32)
        b = rng.standard_normal(128).astype(np.float32)
        c = oracle.cosine_r1(a, b)
        assert c == oracle.cosine_r1(b, a)  # symmetric
        # scaling by 2^k scales dot, ||a||^2 exactly -> bit-identical cosine
        assert c == oracle.cosine_r1(a * 4.0, b)
        assert c == oracle.cosine_r1(a, b * 0.5)
        assert -1.0 <= c <= 1.0


def test_boundary_score_spec_examples():
    # identical -> 1.0; head cosines 1 and 0 -> 0.5; single head [1,0] vs [1,1] -> .7071
    q = np.array([[1.0, 2.0], [3.0, -1.0]], np.float32)
    assert abs(oracle.trigger_r1(q, q, 2, 0.5)[1] - 1.0) < 1e-15
    f, r = oracle.trigger_r1([[1, 0], [1, 0]], [[1, 0], [0, 1]], 2, 0.6)
    assert r == 0.5 and f == 1
    f, r = oracle.trigger_r1([[1, 0]], [[1, 1]], 2, 0.7)
    assert abs(r - 0.70710678) < 1e-6 and f == 0
    # t == 1 always fires
    assert oracle.trigger_r1(q, q, 1, -5.0)[0] == 1
    # tau = -1 never fires after t=1; tau = 1.01 always
    rng = np.random.default_rng(1)
    for _ in range(20):
        a = rng.standard_normal((4, 16)).astype(np.float32)
        b = rng.standard_normal((4, 16)).astype(np.float32)
        assert oracle.trigger_r1(a, b, 3, -1.0)[0] == 0
        assert oracle.trigger_r1(a, b, 3, 1.01)[0] == 1


def test_r_is_mean_of_head_cosines_not_cosine_of_concat():
    # Reading R-AMB2 (P:104 averages per-head cosines). Heads with very different norms:
    a = np.array([[1, 0], [100, 0]], np.float32)
    b = np.array([[0, 1], [100, 0]], np.float32)
    r = oracle.trigger_r1(a, b, 2, 0.0)[1]
    assert r == 0.5  # (0 + 1)/2, whereas the concatenated cosine would be ~0.9999


def test_tau_monotone_boundary_sets_prev_step():
    rng = np.random.default_rng(2)
    qs = rng.standard_normal((40, 4, 8)).astype(np.float32)
    qs[5:12] = qs[5]  # a constant stretch
    taus = [-0.5, 0.0, 0.3, 0.9, 1.01]
    sets = []
    for tau in taus:
        s = {1}
        for t in range(2, 41):
            if oracle.trigger_r1(qs[t - 2], qs[t - 1], t, tau)[0]:
                s.add(t)
        sets.append(s)
    for a, b in zip(sets, sets[1:]):
        assert a <= b


# ---------------------------------------------------------------- exp R3
def test_exp_r3_accuracy_vs_libm():
    x = -np.concatenate([np.linspace(0, 87, 20001), np.logspace(-8, 1.9, 3001)]).astype(np.float32)
    got = oracle.exp_r3(x).astype(np.float64)
    ref = np.exp(x.astype(np.float64))
    rel = np.abs(got - ref) / ref
    # error budget of the recipe: fl32(x*log2e) carries |t|*2^-24 absolute error in the
    # exponent (-> relative |x|*2^-24 in the result), plus ~1.2e-7 Taylor remainder
    # (ln2/2)^7/7! and two fp32 roundings.
    bound = 4e-7 + np.abs(x.astype(np.float64)) * 2.0 ** -24 * 1.1
    assert np.all(rel <= bound)
    assert rel[np.abs(x) < 1].max() < 4e-7
    assert oracle.exp_r3(np.array([0.0], np.float32))[0] == 1.0
    assert oracle.exp_r3(np.array([-200.0], np.float32))[0] == 0.0


# ---------------------------------------------------------------- group scores R2
def test_group_scores_spec_closed_forms():
    # S:340 singleton; S:342 d=1, q=[ln 3], C=[[1],[0]] -> [.75, .25]
    assert oracle.group_scores_r2([[0.3]], [[2.0]])[0] == 1.0
    A = oracle.group_scores_r2([[math.log(3)]], [[1.0], [0.0]])
    assert abs(A[0] - 0.75) < 1e-6 and abs(A[1] - 0.25) < 1e-6
    # d=4: 1/sqrt(d) = 0.5 scale: q=[2ln3,0,0,0] -> logits ln3, 0
    A = oracle.group_scores_r2([[2 * math.log(3), 0, 0, 0]], [[1, 0, 0, 0], [0, 1, 0, 0]])
    assert abs(A[0] - 0.75) < 1e-6


def test_group_scores_identical_heads_equal_g1():
    # S:341 / P:247: g identical heads reduce to per-head retrieval
    rng = np.random.default_rng(3)
    q = rng.standard_normal((1, 128)).astype(np.float32)
    C = rng.standard_normal((300, 128)).astype(np.float32)
    A1 = oracle.group_scores_r2(q, C)
    A4 = oracle.group_scores_r2(np.repeat(q, 4, 0), C)
    assert np.array_equal(A1, A4)


def test_group_scores_sum_to_one_and_match_fp64_definition():
    rng = np.random.default_rng(4)
    for g, n in [(1, 7), (4, 513), (8, 2000)]:
        q = (rng.standard_normal((g, 128)) * 3).astype(np.float32)
        C = (rng.standard_normal((n, 128)) * 2).astype(np.float32)
        A = oracle.group_scores_r2(q, C).astype(np.float64)
        assert abs(A.sum() - 1.0) < 1e-5
        # fp64 check against torch softmax (library definition of the App. B formula)
        import torch
        l = torch.from_numpy(q.astype(np.float64)) @ torch.from_numpy(C.astype(np.float64)).T / math.sqrt(128)
        ref = torch.softmax(l, dim=1).mean(0).numpy()
        # forward error of the fp32 recipe: a d-term fmaf chain errs by at most
        # d*2^-24*sum|q_e c_e| per logit (scaled by 1/sqrt(d)); the softmax turns a logit
        # error into the same relative error (plus the max's), exp_R3 adds ~4e-7.
        el = 128 * 2.0 ** -24 * (np.abs(q).astype(np.float64) @ np.abs(C).astype(np.float64).T) / math.sqrt(128)
        bound = 2 * el.max() + 1e-6
        assert np.max(np.abs(A - ref) / ref) <= bound


def test_group_scores_permutation_equivariant_bitwise():
    rng = np.random.default_rng(5)
    q = rng.standard_normal((4, 128)).astype(np.float32)
    C = rng.standard_normal((257, 128)).astype(np.float32)
    perm = rng.permutation(257)
    A = oracle.group_scores_r2(q, C)
    Ap = oracle.group_scores_r2(q, C[perm])
    assert np.array_equal(A[perm], Ap)  # Z is an exact integer sum: order independent


def test_group_scores_g1_ranking_equals_logit_ranking():
    rng = np.random.default_rng(6)
    q = rng.standard_normal((1, 128)).astype(np.float32)
    C = rng.standard_normal((500, 128)).astype(np.float32)
    A = oracle.group_scores_r2(q, C)
    logits = C.astype(np.float64) @ q[0].astype(np.float64)
    top_a = np.argsort(-A.astype(np.float64), kind="stable")[:50]
    top_l = np.argsort(-logits, kind="stable")[:50]
    assert np.array_equal(top_a, top_l)
