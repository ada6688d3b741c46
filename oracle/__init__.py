"""LouisKV CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct implementation of the LouisKV retrieval hot path
(arXiv 2510.11292), written from PAPER.md. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. The product library
``paper_2510_11292_b200`` never imports it and shares no code with it.

Numerics live in ``louiskv_oracle.c`` (built to ``liblouiskv_oracle.so``);
``episode.py`` sequences them in Algorithm 1's order.
"""
from .core import (  # noqa: F401
    bf16_round,
    e4m3_round,
    cosine_r1,
    trigger_r1,
    exp_r3,
    group_scores_r2,
    group_scores_f64,
    select_greedy,
    kmeans,
    segment_centroid,
    centroids_of,
    attention_f64,
    build_oracle,
)
