"""Retrieval-policy ablation on the C2 synthetic trace with the product kernels (
the paper's system ablation and retrieval-frequency-vs-tau study, P:189, P:446, P:451-465 — here the
efficiency side only: retrievals per layer-step, host-link bytes and decode step time; the accuracy
side needs the paper's models and datasets).

Variants (all on louiskv_decode_layer, graph-replayed 32-layer steps, device-resident inputs):
  * semantic boundary trigger (SR) at tau in {0.5, 0.7, 0.85 (C2), 0.95}, and tau = 2 (per-token);
  * fixed-stride retrieval every 5 / 16 steps (trigger_stride);
  * page units instead of k-means clusters (prompt_units = PAGES: the prompt split on the device into
    contiguous 16-token pages with mean-key centroids), semantic trigger at tau = 0.85.
usage: python tools/ablation.py [--steps 96] > profiles/r01_ablation.json
"""
import argparse, json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np
import torch
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=96)
ap.add_argument("--config", default="C2")
args = ap.parse_args()
base = CONFIGS[args.config]
dev = torch.device("cuda", 0)
VARIANTS = [("SR tau=0.5", 0.5, 0, "kmeans"), ("SR tau=0.7", 0.7, 0, "kmeans"), ("SR tau=0.85", 0.85, 0, "kmeans"),
            ("SR tau=0.95", 0.95, 0, "kmeans"), ("per-token (tau=2)", 2.0, 0, "kmeans"),
            ("fixed stride 5", 0.85, 5, "kmeans"), ("fixed stride 16", 0.85, 16, "kmeans"),
            ("pages of 16, SR tau=0.85", 0.85, 0, "pages")]


res = []
for name, tau, stride, units in VARIANTS:
    cfg = base.replace(tau=tau)
    L, full = cfg.num_layers, set(cfg.full_cache_layers)
    T = 2 + 8 + args.steps
    ctx = lkv.Context(lkv.make_config(cfg, max_output_len=T + 1, trigger_stride=stride,
                                      prompt_units=lkv.UNITS_PAGES if units == "pages" else lkv.UNITS_KMEANS))
    plants = [synth.planted(cfg, l, 0, dev) for l in range(L)]
    for l in range(L):
        K, V = synth.prompt_kv(cfg, l, 0, dev, plants[l])
        ctx.cluster_prompt(l, K, V)
        del K, V
    ctx.prompt_fence()
    q, kk, vv, _ = synth.decode_stream(cfg, T, 0, dev, plants)
    del plants
    q_in, k_in, v_in = q[0].clone(), kk[0].clone(), vv[0].clone()
    out = torch.empty_like(q_in)

    def issue():
        for l in range(L):
            ctx.decode_layer(l, q_in[l], k_in[l], v_in[l], out[l])

    issue()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        issue()
    i = 1
    for _ in range(8):
        q_in.copy_(q[i]); k_in.copy_(kk[i]); v_in.copy_(vv[i]); g.replay(); i += 1
    torch.cuda.synchronize()
    st0 = ctx.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        q_in.copy_(q[i]); k_in.copy_(kk[i]); v_in.copy_(vv[i]); g.replay(); i += 1
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    st1 = ctx.stats()
    d = {k_: st1[k_] - st0[k_] for k_ in st1}
    nrl = (L - len(full)) * cfg.batch
    row = {"variant": name, "tau": tau, "trigger_stride": stride, "units": units, "ms_per_step": ms,
           "tok_per_s": cfg.batch / (ms / 1e3),
           "retrievals_per_layer_step": d["retrievals"] / (args.steps * nrl),
           "h2d_MB_per_step": d["bytes_h2d"] / args.steps / 1e6,
           "reuse_frac": d["units_reused"] / max(d["units_selected"], 1),
           "units_selected_per_retrieval": d["units_selected"] / max(d["retrievals"] * cfg.num_kv_heads, 1)}
    res.append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
    del ctx, g, q, kk, vv
    torch.cuda.empty_cache()
print(json.dumps({"config": cfg.name, "steps": args.steps, "data": "synthetic C2 trace (seed 0)", "rows": res}, indent=1))
