"""Oracle pinned to the worked examples printed in SPEC.md (tests/golden/, each entry cited).

The fixture values are the printed ones; nothing in the fixture was produced by code in this repo.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def _ids(key):
    return [e["cite"] for e in GOLDEN[key]]


@pytest.mark.parametrize("e", GOLDEN["cosine"], ids=_ids("cosine"))
def test_cosine(e):
    assert abs(oracle.cosine_r1(e["a"], e["b"]) - e["expect"]) <= e["tol"]


@pytest.mark.parametrize("e", GOLDEN["boundary_score"], ids=_ids("boundary_score"))
def test_boundary_score(e):
    _, r = oracle.trigger_r1(np.array(e["q_prev"]), np.array(e["q_cur"]), 2, 0.0)
    assert abs(r - e["expect"]) <= e["tol"]


@pytest.mark.parametrize("e", GOLDEN["trigger"], ids=_ids("trigger"))
def test_trigger(e):
    flag, _ = oracle.trigger_r1(np.array(e["q_prev"]), np.array(e["q_cur"]), e["t"], e["tau"])
    assert flag == e["expect"]


@pytest.mark.parametrize("e", GOLDEN["group_scores"], ids=_ids("group_scores"))
def test_group_scores(e):
    q, C = np.array(e["q"]), np.array(e["C"])
    np.testing.assert_allclose(oracle.group_scores_f64(q, C), e["expect"], atol=e["tol"], rtol=0)
    np.testing.assert_allclose(oracle.group_scores_r2(q, C), e["expect"], atol=max(e["tol"], 1e-6), rtol=0)


@pytest.mark.parametrize("e", GOLDEN["select_units"], ids=_ids("select_units"))
def test_select_units(e):
    assert sorted(oracle.select_greedy(e["scores"], e["sizes"], e["B"]).tolist()) == e["expect"]


@pytest.mark.parametrize("e", GOLDEN["centroid"], ids=_ids("centroid"))
def test_centroid(e):
    np.testing.assert_allclose(oracle.segment_centroid(np.array(e["keys"])), e["expect"], atol=e["tol"] + 1e-7, rtol=0)


@pytest.mark.parametrize("e", GOLDEN["attention"], ids=_ids("attention"))
def test_attention(e):
    out = oracle.attention_f64(np.array(e["q"]), np.array(e["K"]), np.array(e["V"]))
    np.testing.assert_allclose(out[0], e["expect"], atol=e["tol"] + 1e-7, rtol=0)


@pytest.mark.parametrize("e", GOLDEN["kmeans_k"], ids=_ids("kmeans_k"))
def test_kmeans_cluster_count(e):
    k = math.ceil(e["n"] / e["c"])
    assert k == e["expect_k"]
    rng = np.random.default_rng(0)
    X = rng.standard_normal((e["n"], 4)).astype(np.float32)
    _, _, counts, _, _ = oracle.kmeans(X, k, 10)
    assert counts.sum() == e["n"] and (counts >= 1).all()
