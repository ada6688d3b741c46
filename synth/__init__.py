"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the LouisKV method: it only draws random
tensors with the structure of the paper's workloads (DESIGN.md §Input recipe):

* prompt keys: ``x_i = mu0 + mu_{c(i)} + 0.5 N(0,I)`` with ``k_pl`` planted
  directions ``mu_c ~ 2 N(0,I)`` scattered over positions — the "sparse"
  input layout of Observation 2;
* values ``N(0,I)``;
* decode queries in segments of geometric length (mean 5 for long-input, 16
  for long-output, matching the fixed-stride equivalence of P:446); inside a
  segment, query head h aims at a target set T_j of 8 planted directions of
  its KV head; T_{j+1} keeps half of T_j; per-step noise keeps the
  within-segment cosine near 0.95 (Observation 1);
* decode keys ``k_t = mu0 + w_j + 0.5 N(0,I)`` per segment — the "dense"
  output layout.

Everything is bf16 (RNE via torch's cast). Generation runs with torch on any
device; both sides receive the very same tensors.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import torch

from .configs import Config, CONFIGS  # noqa: F401


def _gen(device, *key) -> torch.Generator:
    h = 1469598103934665603
    for k in key:
        h = ((h ^ (int(k) & 0xFFFFFFFFFFFF)) * 1099511628211) & 0x7FFFFFFFFFFFFFFF
    g = torch.Generator(device=device)
    g.manual_seed(h)
    return g


def _randn(shape, g, device, scale=1.0):
    return torch.randn(shape, generator=g, device=device, dtype=torch.float32) * scale


@dataclasses.dataclass
class LayerPlant:
    mu0: torch.Tensor        # [b, Hkv, d] fp32
    mu: torch.Tensor         # [b, Hkv, k_pl, d] fp32 planted directions


def planted(cfg: Config, layer: int, seed: int, device="cpu") -> LayerPlant:
    g = _gen(device, seed, 1, layer)
    b, H, d = cfg.batch, cfg.num_kv_heads, cfg.head_dim
    mu0 = _randn((b, H, d), g, device)
    mu = _randn((b, H, cfg.k_planted, d), g, device, 2.0)
    return LayerPlant(mu0, mu)


def prompt_kv(cfg: Config, layer: int, seed: int, device="cpu", plant: Optional[LayerPlant] = None,
              layout: str = "scattered", return_labels: bool = False):
    """K, V bf16 [b, P, Hkv, d] for one layer.

    layout="scattered": each position draws its planted group at random (the sparse input
    layout of P:90); layout="blocked": group j occupies positions [S + j*N/k_pl, ...), so
    the strided k-means init seeds one centroid per group (well-separated parity inputs).
    With return_labels, also returns the planted group id per (b, position, head)."""
    if plant is None:
        plant = planted(cfg, layer, seed, device)
    g = _gen(device, seed, 2, layer)
    b, P, H, d = cfg.batch, cfg.prompt_len, cfg.num_kv_heads, cfg.head_dim
    if layout == "blocked":
        S = min(cfg.sink_tokens, P)
        N = P - S
        pos = torch.arange(P, device=device)
        grp = torch.clamp(((pos - S).clamp(min=0) * cfg.k_planted) // max(N, 1), max=cfg.k_planted - 1)
        cid = grp.view(1, P, 1).expand(b, P, H).contiguous()
        _ = torch.randint(0, 2, (1,), generator=g, device=device)
    else:
        cid = torch.randint(0, cfg.k_planted, (b, P, H), generator=g, device=device)
    # gather planted direction per (b, pos, head)
    mu = plant.mu  # [b, H, k, d]
    idx = cid.permute(0, 2, 1)  # [b, H, P]
    sel = torch.gather(mu, 2, idx.unsqueeze(-1).expand(b, H, P, d))  # [b, H, P, d]
    K = plant.mu0.unsqueeze(2) + sel + _randn((b, H, P, d), g, device, cfg.key_noise)
    K = K.permute(0, 2, 1, 3).contiguous()
    V = _randn((b, P, H, d), g, device)
    if return_labels:
        return K.to(torch.bfloat16), V.to(torch.bfloat16), cid
    return K.to(torch.bfloat16), V.to(torch.bfloat16)


def segment_lengths(cfg: Config, steps: int, seed: int, b: int):
    """Geometric segment lengths (mean cfg.seg_mean) covering `steps` steps."""
    g = _gen("cpu", seed, 3, b)
    p = 1.0 / cfg.seg_mean
    lens, tot = [], 0
    while tot < steps:
        u = torch.rand((), generator=g).item()
        n = 1 + int(math.floor(math.log(max(1.0 - u, 1e-12)) / math.log(1.0 - p))) if p < 1 else 1
        lens.append(n)
        tot += n
    return lens


def boundaries(cfg: Config, steps: int, seed: int):
    """Planted segment-start steps (1-based) per sequence b: list of sets."""
    out = []
    for b in range(cfg.batch):
        s, t = set(), 1
        for n in segment_lengths(cfg, steps, seed, b):
            s.add(t)
            t += n
        out.append(s)
    return out


def decode_stream(cfg: Config, steps: int, seed: int, device="cpu", plants=None, rho: float = 0.5):
    """Per-step decode inputs for all layers.

    Returns q [steps, L, b, Hq, d], k, v [steps, L, b, Hkv, d] (bf16) and the
    planted boundary sets.
    """
    L, b, Hq, Hkv, d = cfg.num_layers, cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
    gq = cfg.group
    q = torch.empty((steps, L, b, Hq, d), dtype=torch.bfloat16, device=device)
    k = torch.empty((steps, L, b, Hkv, d), dtype=torch.bfloat16, device=device)
    v = torch.empty((steps, L, b, Hkv, d), dtype=torch.bfloat16, device=device)
    seg_lens = [segment_lengths(cfg, steps, seed, bb) for bb in range(b)]
    kvmap = torch.arange(Hq) // gq
    for layer in range(L):
        plant = plants[layer] if plants is not None else planted(cfg, layer, seed, device)
        g = _gen(device, seed, 4, layer)
        gc = _gen("cpu", seed, 5, layer)
        mu = plant.mu  # [b, Hkv, k, d]
        unit = mu / mu.norm(dim=-1, keepdim=True)
        nt, kp = cfg.n_targets, cfg.k_planted
        for bb in range(b):
            t0 = 0
            targets = torch.stack([torch.randperm(kp, generator=gc)[:nt] for _ in range(Hkv)])  # [Hkv, nt]
            for j, n in enumerate(seg_lens[bb]):
                n_eff = min(n, steps - t0)
                if n_eff <= 0:
                    break
                if j > 0:
                    keep = int(round(rho * nt))
                    new_t = []
                    for h in range(Hkv):
                        old = targets[h][torch.randperm(nt, generator=gc)[:keep]].tolist()
                        chosen, taken = list(old), set(old)
                        while len(chosen) < nt:
                            c = int(torch.randint(0, kp, (1,), generator=gc))
                            if c not in taken:
                                taken.add(c)
                                chosen.append(c)
                        new_t.append(torch.tensor(chosen))
                    targets = torch.stack(new_t)
                # query directions per q head: weighted sum of its KV head's target directions
                w = (0.5 + torch.rand((Hq, nt), generator=gc)).to(device)
                tg = targets[kvmap].to(device)                       # [Hq, nt]
                dirs = unit[bb][kvmap.to(device).unsqueeze(1), tg]   # [Hq, nt, d]
                u = (w.unsqueeze(-1) * dirs).sum(1)
                u = u / u.norm(dim=-1, keepdim=True) * cfg.q_scale
                noise = _randn((n_eff, Hq, d), g, device, cfg.q_noise * cfg.q_scale)
                if cfg.drift > 0:
                    # graded drift: the direction random-walks inside the segment with a per-segment
                    # step size, so consecutive-query cosines spread over a range instead of one value
                    step = float(torch.rand((), generator=gc)) * cfg.drift * cfg.q_scale / math.sqrt(d)
                    walk = torch.cumsum(_randn((n_eff, Hq, d), g, device, step), dim=0)
                    uu = u.unsqueeze(0) + walk
                    uu = uu / uu.norm(dim=-1, keepdim=True) * cfg.q_scale
                    q[t0:t0 + n_eff, layer, bb] = (uu + noise).to(torch.bfloat16)
                else:
                    q[t0:t0 + n_eff, layer, bb] = (u.unsqueeze(0) + noise).to(torch.bfloat16)
                wdir = _randn((Hkv, d), g, device, 2.0)
                kk = plant.mu0[bb].unsqueeze(0) + wdir.unsqueeze(0) + _randn((n_eff, Hkv, d), g, device, cfg.key_noise)
                k[t0:t0 + n_eff, layer, bb] = kk.to(torch.bfloat16)
                v[t0:t0 + n_eff, layer, bb] = _randn((n_eff, Hkv, d), g, device).to(torch.bfloat16)
                t0 += n_eff
    bset = []
    for bb in range(b):
        s, t = set(), 1
        for n in seg_lens[bb]:
            if t > steps:
                break
            s.add(t)
            t += n
        bset.append(s)
    return q, k, v, bset
