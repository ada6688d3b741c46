"""Algorithm 1 on the CPU — TEST INFRASTRUCTURE ONLY.

Sequences the oracle primitives of ``louiskv_oracle.c`` in the paper's order.
Python here only does bookkeeping (lists, sets, slicing); every arithmetic
step (cosine, k-means, centroid, scores, selection, attention) is a call into
the C oracle. Readings of silent passages are DESIGN.md §Readings.

Per decode step t and layer:
  1. r_t / flag                      -> should_retrieve
  2. if flag: score all host units, select under B,      -> retrieve
     load them
  3. store_cache(k_t, v_t, 'decode')  -> append_output
  4. attention over [sinks : KV_critical : KV_local]     -> sparse_attn
     (P:143); full-cache layers attend to everything.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional

import numpy as np

from . import core

PREV_STEP, LAST_RETRIEVAL = 0, 1
PER_LAYER, SHARED = 0, 1


@dataclasses.dataclass
class Unit:
    uid: int
    positions: np.ndarray      # token positions (ascending)
    K: np.ndarray              # [n, d] fp32 (bf16 values)
    V: np.ndarray
    centroid: np.ndarray       # fp32 [d]
    centroid_bf16: np.ndarray  # fp32 [d] holding bf16 values


class _Inst:
    """State of one (layer, b, kv-head) instance of a retrieval layer."""

    def __init__(self):
        self.sinks_K = None
        self.sinks_V = None
        self.units: List[Unit] = []
        self.selected: List[int] = []      # working set: unit ids ascending
        self.open_K: List[np.ndarray] = []  # open segment rows
        self.open_V: List[np.ndarray] = []
        self.open_pos: List[int] = []
        self.sealed: List[dict] = []       # FIFO of sealed segments in the local buffer


class OracleEpisode:
    def __init__(self, cfg, trigger_ref=PREV_STEP, boundary_mode=PER_LAYER, shared_layer=0,
                 max_open_segment: Optional[int] = None, kmeans_mode: int = 1,
                 kv_head_begin: int = 0, kv_head_count: Optional[int] = None, trigger_stride: int = 0,
                 pool_fp8: bool = False):
        self.cfg = cfg
        # trigger_stride k >= 1: the fixed-stride retrieval of the paper's ablation — retrieve
        # at t = 1, 1 + k, 1 + 2k, ... instead of on r_t < tau; 0: the semantic boundary
        self.stride = int(trigger_stride)
        self.L, self.Hq, self.Hkv, self.d = cfg.num_layers, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim
        self.g = self.Hq // self.Hkv
        self.b = cfg.batch
        self.S, self.W, self.B, self.tau = cfg.sink_tokens, cfg.window_tokens, cfg.budget_tokens, cfg.tau
        self.c, self.iters = cfg.avg_cluster_size, cfg.kmeans_iters
        self.full = set(cfg.full_cache_layers)
        self.trigger_ref, self.boundary_mode, self.shared_layer = trigger_ref, boundary_mode, shared_layer
        self.max_open = max_open_segment if max_open_segment is not None else cfg.window_tokens
        self.kmeans_mode = kmeans_mode
        self.h0 = kv_head_begin
        self.hn = kv_head_count if kv_head_count is not None else self.Hkv
        self.P: Dict[int, int] = {}
        self.t: Dict[int, int] = {l: 0 for l in range(self.L)}
        self.q_ref = {l: np.zeros((self.b, self.Hq, self.d), np.float32) for l in range(self.L)}
        self.flags = {l: np.zeros(self.b, np.int32) for l in range(self.L)}
        self.r = {l: np.zeros(self.b, np.float64) for l in range(self.L)}
        self.inst: Dict[tuple, _Inst] = {}
        self.full_K: Dict[tuple, np.ndarray] = {}
        self.full_V: Dict[tuple, np.ndarray] = {}
        self.kmeans_J: Dict[tuple, np.ndarray] = {}
        self.stats = dict(retrievals=0, units_scored=0, units_selected=0, units_reused=0,
                          units_fetched=0, bytes_h2d=0, bytes_d2h=0, segments_evicted=0)
        # pool_fp8 (reading R-FP8, the FP8 host-pool variant of SURVEY §8(f) row 3): every K/V row that
        # enters the CPU pool is stored as E4M3 (RNE, saturating), so a unit's rows — the ones
        # retrieval brings back — are the E4M3 values; sinks and the local buffer stay bf16, centroids
        # are computed from the bf16 keys
        self.pool_fp8 = bool(pool_fp8)
        self.row_bytes = 2 * (1 if self.pool_fp8 else 2) * self.d  # K+V per token per head in the pool

    def _pool(self, x: np.ndarray) -> np.ndarray:
        return core.e4m3_round(x) if self.pool_fp8 else x

    # --------------------------------------------------------------- prefill
    def cluster_prompt(self, layer: int, K: np.ndarray, V: np.ndarray, assign: Optional[np.ndarray] = None):
        """store_cache(K, V, 'prefill'). K, V: [b, P, Hkv_owned, d] fp32.

        ``assign`` ([b, Hkv_owned, P-S] cluster ids) replaces the k-means step with a given
        clustering (centroids are still the means of the members)."""
        K = np.asarray(K, np.float32)
        V = np.asarray(V, np.float32)
        b, P, H, d = K.shape
        self.P[layer] = P
        for bb in range(b):
            for hh in range(H):
                key = (layer, bb, hh)
                if layer in self.full:
                    self.full_K[key] = [K[bb, p, hh].copy() for p in range(P)]
                    self.full_V[key] = [V[bb, p, hh].copy() for p in range(P)]
                    continue
                inst = _Inst()
                S = min(self.S, P)
                inst.sinks_K, inst.sinks_V = K[bb, :S, hh].copy(), V[bb, :S, hh].copy()
                N = P - S
                if N > 0:
                    k = self.cfg.n_clusters if self.cfg.clusters_override else -(-N // self.c)
                    k = min(k, N)
                    X = K[bb, S:, hh]
                    if assign is None:
                        a_i, C, counts, J, _ = core.kmeans(X, k, self.iters, self.kmeans_mode)
                        self.kmeans_J[key] = J
                    else:
                        a_i = np.asarray(assign[bb, hh], np.int32)
                        C = core.centroids_of(X, a_i, k)
                    Cb = core.bf16_round(C)
                    for j in range(k):
                        mem = np.nonzero(a_i == j)[0]
                        inst.units.append(Unit(j, mem + S, self._pool(X[mem]), self._pool(V[bb, S + mem, hh]),
                                               C[j].copy(), Cb[j].copy()))
                    self.stats["bytes_d2h"] += N * self.row_bytes
                self.inst[key] = inst

    # ---------------------------------------------------------------- decode
    def should_retrieve(self, layer: int, q_all: np.ndarray):
        """r_t and flag per sequence (Alg. 1). q_all [b, Hq, d]."""
        q_all = np.asarray(q_all, np.float32)
        self.t[layer] += 1
        t = self.t[layer]
        if layer in self.full:
            self.flags[layer][:] = 0
            return self.flags[layer].copy(), self.r[layer].copy()
        if self.boundary_mode == SHARED and layer != self.shared_layer:
            self.flags[layer][:] = self.flags[self.shared_layer]
            self.r[layer][:] = self.r[self.shared_layer]
            return self.flags[layer].copy(), self.r[layer].copy()
        for bb in range(self.b):
            f, r = core.trigger_r1(self.q_ref[layer][bb], q_all[bb], t, self.tau)
            if self.stride > 0:
                f = 1 if (t - 1) % self.stride == 0 else 0
            self.flags[layer][bb], self.r[layer][bb] = f, r
            if self.trigger_ref == PREV_STEP or f:
                self.q_ref[layer][bb] = q_all[bb]
        return self.flags[layer].copy(), self.r[layer].copy()

    def retrieve(self, layer: int, q_own: np.ndarray):
        """kvm.retrieve(q_t, B) for flagged sequences. q_own [b, g*Hkv_owned, d]."""
        if layer in self.full:
            return
        q_own = np.asarray(q_own, np.float32)
        for bb in range(self.b):
            if not self.flags[layer][bb]:
                continue
            self.stats["retrievals"] += 1
            for hh in range(self.hn):
                inst = self.inst[(layer, bb, hh)]
                n = len(inst.units)
                if n == 0:
                    new_sel = []
                else:
                    Cb = np.stack([u.centroid_bf16 for u in inst.units])
                    A = core.group_scores_r2(q_own[bb, hh * self.g:(hh + 1) * self.g], Cb)
                    sizes = np.array([u.positions.size for u in inst.units], np.int32)
                    new_sel = core.select_greedy(A, sizes, self.B).tolist()
                    self.stats["units_scored"] += n
                old = set(inst.selected)
                for u in new_sel:
                    if u in old:
                        self.stats["units_reused"] += 1
                    else:
                        self.stats["units_fetched"] += 1
                        self.stats["bytes_h2d"] += inst.units[u].positions.size * self.row_bytes
                self.stats["units_selected"] += len(new_sel)
                inst.selected = new_sel

    def append_output(self, layer: int, k_t: np.ndarray, v_t: np.ndarray):
        """store_cache(k_t, v_t, 'decode'). k_t, v_t [b, Hkv_owned, d]."""
        k_t = np.asarray(k_t, np.float32)
        v_t = np.asarray(v_t, np.float32)
        t = self.t[layer]
        P = self.P[layer]
        pos = P + t - 1
        for bb in range(self.b):
            for hh in range(self.hn):
                key = (layer, bb, hh)
                if layer in self.full:
                    self.full_K[key].append(k_t[bb, hh].copy())
                    self.full_V[key].append(v_t[bb, hh].copy())
                    continue
                inst = self.inst[key]
                flag = self.flags[layer][bb]
                n_open = len(inst.open_pos)
                # seal the open segment at a boundary or at the force-seal bound (R-AMB13)
                if (flag and n_open > 0) or n_open >= self.max_open:
                    Ko = np.stack(inst.open_K)
                    cen = core.segment_centroid(Ko)
                    inst.sealed.append(dict(K=Ko, V=np.stack(inst.open_V),
                                            pos=np.array(inst.open_pos, np.int64), centroid=cen))
                    inst.open_K, inst.open_V, inst.open_pos = [], [], []
                inst.open_K.append(k_t[bb, hh].copy())
                inst.open_V.append(v_t[bb, hh].copy())
                inst.open_pos.append(pos)
                # evict the oldest sealed segment while the buffer holds more than W tokens
                while inst.sealed and (sum(s["pos"].size for s in inst.sealed) + len(inst.open_pos)) > self.W:
                    s = inst.sealed.pop(0)
                    uid = len(inst.units)
                    inst.units.append(Unit(uid, s["pos"], self._pool(s["K"]), self._pool(s["V"]), s["centroid"],
                                           core.bf16_round(s["centroid"])))
                    self.stats["bytes_d2h"] += s["pos"].size * self.row_bytes
                    self.stats["segments_evicted"] += 1

    def attention_rows(self, layer: int, bb: int, hh: int):
        """(positions, K, V) of the attention set [sinks : critical : local]."""
        key = (layer, bb, hh)
        if layer in self.full:
            K = np.stack(self.full_K[key])
            V = np.stack(self.full_V[key])
            return np.arange(K.shape[0]), K, V
        inst = self.inst[key]
        pos = [np.arange(inst.sinks_K.shape[0])]
        Ks, Vs = [inst.sinks_K], [inst.sinks_V]
        for u in inst.selected:
            U = inst.units[u]
            pos.append(U.positions)
            Ks.append(U.K)
            Vs.append(U.V)
        for s in inst.sealed:
            pos.append(s["pos"])
            Ks.append(s["K"])
            Vs.append(s["V"])
        if inst.open_pos:
            pos.append(np.array(inst.open_pos))
            Ks.append(np.stack(inst.open_K))
            Vs.append(np.stack(inst.open_V))
        return np.concatenate(pos), np.concatenate(Ks), np.concatenate(Vs)

    def sparse_attn(self, layer: int, q_own: np.ndarray) -> np.ndarray:
        """o = softmax(q K_I^T/sqrt(d)) V_I per query head. fp64 [b, g*Hkv_owned, d]."""
        q_own = np.asarray(q_own, np.float32)
        out = np.zeros((self.b, self.g * self.hn, self.d), np.float64)
        for bb in range(self.b):
            for hh in range(self.hn):
                _, K, V = self.attention_rows(layer, bb, hh)
                qg = q_own[bb, hh * self.g:(hh + 1) * self.g]
                out[bb, hh * self.g:(hh + 1) * self.g] = core.attention_f64(qg, K, V)
        return out

    # ---------------------------------------------------------------- helpers
    def units(self, layer: int, bb: int, hh: int) -> List[Unit]:
        return self.inst[(layer, bb, hh)].units

    def selection(self, layer: int, bb: int, hh: int) -> List[int]:
        return list(self.inst[(layer, bb, hh)].selected)

    def step(self, q_all, k_t, v_t):
        """One decode step over all layers in model order. q_all [L, b, Hq, d]."""
        outs = []
        for layer in range(self.L):
            qa = np.asarray(q_all[layer], np.float32)
            self.should_retrieve(layer, qa)
            qo = qa[:, self.h0 * self.g:(self.h0 + self.hn) * self.g]
            self.retrieve(layer, qo)
            self.append_output(layer, k_t[layer][:, self.h0:self.h0 + self.hn], v_t[layer][:, self.h0:self.h0 + self.hn])
            outs.append(self.sparse_attn(layer, qo))
        return np.stack(outs)
