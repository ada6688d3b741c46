"""Run the CUDA path (through the C ABI) and the oracle side by side on the same
seeded inputs. Shared by the -m gpu parity tests, smoke() and bench.py."""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np
import torch

import oracle
import synth
from oracle.episode import OracleEpisode


def bf16_bits(x_f32: np.ndarray) -> np.ndarray:
    """bf16 bit pattern of fp32 arrays that hold exact bf16 values."""
    return (np.ascontiguousarray(x_f32, np.float32).view(np.uint32) >> 16).astype(np.uint16)


@dataclasses.dataclass
class Inputs:
    K: List[torch.Tensor]    # per layer [b, P, Hkv, d] bf16 (cuda)
    V: List[torch.Tensor]
    labels: List[torch.Tensor]
    q: torch.Tensor          # [T, L, b, Hq, d]
    k: torch.Tensor          # [T, L, b, Hkv, d]
    v: torch.Tensor
    bset: list


def make_inputs(cfg, steps, seed, device="cuda", layout="scattered") -> Inputs:
    plants = [synth.planted(cfg, l, seed, device) for l in range(cfg.num_layers)]
    K, V, lab = [], [], []
    for l in range(cfg.num_layers):
        a, b_, c = synth.prompt_kv(cfg, l, seed, device, plants[l], layout=layout, return_labels=True)
        K.append(a)
        V.append(b_)
        lab.append(c)
    q, k, v, bset = synth.decode_stream(cfg, steps, seed, device, plants)
    return Inputs(K, V, lab, q, k, v, bset)


def np32(t: torch.Tensor) -> np.ndarray:
    return t.float().cpu().numpy()


def oracle_assign(cfg, K_np: np.ndarray, mode: int = 1) -> np.ndarray:
    """Oracle k-means assignment [b, H, N] of one layer (for injection into both sides)."""
    b, P, H, d = K_np.shape
    S = min(cfg.sink_tokens, P)
    N = P - S
    k = -(-N // cfg.avg_cluster_size)
    out = np.zeros((b, H, N), np.int32)
    for bb in range(b):
        for hh in range(H):
            out[bb, hh] = oracle.kmeans(K_np[bb, S:, hh], k, cfg.kmeans_iters, mode)[0]
    return out


def planted_assign(cfg, labels: torch.Tensor) -> np.ndarray:
    """Planted labels as a clustering of [S, P) with every cluster non-empty."""
    lab = labels.cpu().numpy()  # [b, P, H]
    b, P, H = lab.shape
    S = min(cfg.sink_tokens, P)
    N = P - S
    k = -(-N // cfg.avg_cluster_size)
    a = (lab[:, S:, :].transpose(0, 2, 1) % k).astype(np.int32).copy()
    a[:, :, :k] = np.arange(k, dtype=np.int32)
    return a
