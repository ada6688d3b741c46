"""Workload configurations (BASELINE.json ``configs``).

Numbers only — no method arithmetic. Paper parameters: S, W, tau per task
family (P:148 long-input: S=32, W=512, tau=0.85; P:150 long-output: S=500 or
64, W=128 or 256, tau=0.7), average cluster size c=16 and two full-cache layers
(P:143), budgets 512 / 1024. Model shapes not in the paper come
from the public model configs (Llama-3.1-8B: 32 layers, 32 q heads, 8 KV heads;
Qwen3-8B: 36/32/8; Qwen3-32B: 64/64/8; all d=128).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Tuple


@dataclasses.dataclass
class Config:
    name: str
    num_layers: int
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    batch: int
    prompt_len: int
    decode_steps: int
    sink_tokens: int
    window_tokens: int
    budget_tokens: int
    tau: float
    avg_cluster_size: int
    kmeans_iters: int = 10
    full_cache_layers: Tuple[int, ...] = (0, 1)
    seg_mean: float = 5.0
    # generator knobs (DESIGN.md §Input recipe)
    k_planted: int = 0          # 0 -> k (well separated, parity) ; set k//4 for throughput
    key_noise: float = 0.5
    n_targets: int = 8
    q_scale: float = 6.0
    q_noise: float = 0.0203     # per-coordinate sigma relative to |u| (within-segment cos ~0.95)
    max_output_len: int = 0     # 0 -> decode_steps
    drift: float = 0.0          # > 0: graded within-segment query drift (random walk of the direction,
                                # per-segment step size uniform in [0, drift] x |u|): spreads r_t so a
                                # tau sweep traces a retrieval-frequency curve (ablation inputs only)
    clusters_override: int = 0  # C1: k fixed at 64

    def __post_init__(self):
        if self.k_planted == 0:
            self.k_planted = max(self.n_clusters, self.n_targets * 2)
        if self.max_output_len == 0:
            self.max_output_len = self.decode_steps

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def n_clustered(self) -> int:
        return max(0, self.prompt_len - self.sink_tokens)

    @property
    def n_clusters(self) -> int:
        if self.n_clustered == 0:
            return 0
        if self.clusters_override:
            return self.clusters_override
        return math.ceil(self.n_clustered / self.avg_cluster_size)

    @property
    def full_mask(self) -> int:
        m = 0
        for l in self.full_cache_layers:
            m |= 1 << l
        return m

    def replace(self, **kw) -> "Config":
        d = dataclasses.asdict(self)
        d.update(kw)
        if "k_planted" not in kw:
            d["k_planted"] = 0
        return Config(**d)


# C1: single KV head, 4096-token prompt, 64 clusters, 10 iters, 16 decode steps.
C1 = Config("C1", num_layers=1, num_q_heads=1, num_kv_heads=1, head_dim=128, batch=1,
            prompt_len=4096, decode_steps=16, sink_tokens=0, window_tokens=512, budget_tokens=512,
            tau=0.85, avg_cluster_size=64, clusters_override=64, full_cache_layers=(), seg_mean=5.0)
# C2: Llama-3.1-8B shape, 32K prompt, 512 output, batch 1 (long-input).
C2 = Config("C2", num_layers=32, num_q_heads=32, num_kv_heads=8, head_dim=128, batch=1,
            prompt_len=32768, decode_steps=512, sink_tokens=32, window_tokens=512, budget_tokens=512,
            tau=0.85, avg_cluster_size=16, seg_mean=5.0)
# C3: Qwen3-8B shape, 1K prompt, 32K generated (short-input long-output).
C3 = Config("C3", num_layers=36, num_q_heads=32, num_kv_heads=8, head_dim=128, batch=1,
            prompt_len=1024, decode_steps=32768, sink_tokens=500, window_tokens=128, budget_tokens=1024,
            tau=0.7, avg_cluster_size=16, seg_mean=16.0)
# C4: Qwen3-8B, 64K + 16K, batch 8 (long-input long-output).
C4 = Config("C4", num_layers=36, num_q_heads=32, num_kv_heads=8, head_dim=128, batch=8,
            prompt_len=65536, decode_steps=16384, sink_tokens=64, window_tokens=256, budget_tokens=1024,
            tau=0.7, avg_cluster_size=16, seg_mean=16.0)
# C5: Qwen3-32B, 128K, batch 32 (8 GPUs by KV head).
C5 = Config("C5", num_layers=64, num_q_heads=64, num_kv_heads=8, head_dim=128, batch=32,
            prompt_len=131072, decode_steps=1024, sink_tokens=64, window_tokens=256, budget_tokens=1024,
            tau=0.7, avg_cluster_size=16, seg_mean=16.0)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}
