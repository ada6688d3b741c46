"""Retrieval-policy and system ablations on the product kernels (the paper's system
ablation, and its retrieval-frequency / latency vs tau study, P:451-465 — the efficiency side
only: the accuracy side needs the paper's models and datasets).

Workload: Qwen3-8B long-input long-output shape (36 layers, 32 q heads, 8 KV heads, layers 0-1 full
cache, S=64 W=256 B=1024 c=16) at a 32K prompt and batch 2 (the paper's ablation runs
Qwen3-8B 32K+16K), decode steps graph-replayed with device-resident inputs.

1. System ladder ("we incrementally apply each optimization on top of a baseline system"):
   * base   — retrieval at EVERY decode step (tau = 2 > 1), per-head selection: each query head selects
              its own units (re-created by giving every query head its own copy of its group's KV —
              g = 1, the reduction of group-consistent selection named at P:247), the four-call
              kernel sequence (trigger+logits / select / gather+append / attention);
   * +SR    — the semantic-boundary trigger at tau = 0.7;
   * +GS    — group-consistent selection: one selection per KV head from the g-head mean of the
              softmax scores (App. B), no KV copies;
   * +CK    — the custom single-launch retrieval kernel (louiskv_decode_layer) instead of the
              four-call sequence. (The paper's non-CK baseline is PyTorch; ours is the unfused CUDA
              sequence, so this step measures fusion only.)
2. tau sweep on a graded-drift query generator (synth drift > 0: per-segment random-walk queries, so
   r_t spreads and the retrieval frequency traces a curve): tau in {0.3 .. 0.95}.
3. Fixed-stride retrieval every 5 / 16 steps and 16-token pages at tau = 0.7.
4. Gather variant (§4.3: the paper moves selected rows with DGL's row transfer): the default
   zero-copy gather vs fetch_mode BATCHED_DMA (copy-engine copies, one per merged span, host-issued
   after a stream sync), both through the four-call sequence launched eagerly (BATCHED_DMA cannot be
   graph-captured), on the C2 headline shape (--only fetch).
5. Index placement (the paper's future work: "offloading KV cache indices to CPU DRAM"): the
   unit index (centroids) in device memory vs in pinned host memory read over the link at every
   scoring, C2 and the C4 shape at 32K: step time and device bytes (--only index).
6. Pool element type: bf16 (the paper's) vs E4M3 host pool — half the offload
   and gather bytes; C2 and the C4 shape at 32K (--only fp8).

usage: python tools/ablation.py [--steps 64] > profiles/r02_ablation.json
"""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch

import paper_2510_11292_b200 as lkv
import synth
from synth.configs import C2, C4

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--prompt", type=int, default=32768)
ap.add_argument("--batch", type=int, default=2)
ap.add_argument("--only", default="")
args = ap.parse_args()
BASE = C4.replace(prompt_len=args.prompt, batch=args.batch)
BASE = BASE.replace(k_planted=max(BASE.n_clusters // 4, 16))
dev = torch.device("cuda", 0)


def run(name, cfg, *, per_head=False, fused=True, stride=0, units="kmeans", fetch=0, graph=True, index_offload=0,
        pool_dtype=0):
    """One variant: prefill every layer, warm up, time args.steps decode steps (graph-replayed, or
    issued eagerly with graph=False)."""
    L, full, b = cfg.num_layers, set(cfg.full_cache_layers), cfg.batch
    g = cfg.group
    run_cfg = cfg.replace(num_kv_heads=cfg.num_q_heads, k_planted=cfg.k_planted) if per_head else cfg
    T = 2 + 8 + args.steps
    ctx = lkv.Context(lkv.make_config(run_cfg, max_output_len=T + 1, trigger_stride=stride,
                                      prompt_units=lkv.UNITS_PAGES if units == "pages" else lkv.UNITS_KMEANS,
                                      fetch_mode=fetch, index_offload=index_offload, pool_dtype=pool_dtype))
    plants = [synth.planted(cfg, l, 0, dev) for l in range(L)]
    for l in range(L):
        K, V = synth.prompt_kv(cfg, l, 0, dev, plants[l])
        if per_head:  # every query head its own copy of its group's KV (g = 1)
            K, V = K.repeat_interleave(g, dim=2), V.repeat_interleave(g, dim=2)
        ctx.cluster_prompt(l, K, V)
        del K, V
    ctx.prompt_fence()
    q, kk, vv, _ = synth.decode_stream(cfg, T, 0, dev, plants)
    del plants
    if per_head:
        kk, vv = kk.repeat_interleave(g, dim=3), vv.repeat_interleave(g, dim=3)
    q_in, k_in, v_in = q[0].clone(), kk[0].clone(), vv[0].clone()
    out = torch.empty_like(q_in)

    def issue():
        for l in range(L):
            if fused:
                ctx.decode_layer(l, q_in[l], k_in[l], v_in[l], out[l])
            else:
                ctx.should_retrieve(l, q_in[l])
                ctx.retrieve(l, q_in[l])
                ctx.append_output(l, k_in[l], v_in[l])
                ctx.sparse_attn(l, q_in[l], out[l])

    issue()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    if graph:
        with torch.cuda.graph(gr, stream=s):
            issue()
    else:
        gr.replay = issue
    i = 1
    for _ in range(8):
        q_in.copy_(q[i]); k_in.copy_(kk[i]); v_in.copy_(vv[i]); gr.replay(); i += 1
    torch.cuda.synchronize()
    st0 = ctx.stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        q_in.copy_(q[i]); k_in.copy_(kk[i]); v_in.copy_(vv[i]); gr.replay(); i += 1
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    st1 = ctx.stats()
    d = {k_: st1[k_] - st0[k_] for k_ in st1}
    nrl = (L - len(full)) * b
    row = {"variant": name, "tau": cfg.tau, "drift": cfg.drift, "per_head": per_head, "fused": fused,
           "trigger_stride": stride, "units": units, "fetch": ["zero_copy", "batched_dma"][fetch],
           "graph": graph, "index_offload": index_offload, "pool": ["bf16", "e4m3"][pool_dtype], "memory": ctx.memory(), "ms_per_step": ms, "tok_per_s": b / (ms / 1e3),
           "retrievals_per_layer_step": d["retrievals"] / (args.steps * nrl),
           "h2d_MB_per_step": d["bytes_h2d"] / args.steps / 1e6,
           "reuse_frac": d["units_reused"] / max(d["units_selected"], 1)}
    print(json.dumps(row), file=sys.stderr, flush=True)
    del ctx, gr, q, kk, vv
    torch.cuda.empty_cache()
    return row


rows = {"ladder": [], "tau_sweep": [], "policies": []}
if args.only in ("", "ladder"):
    rows["ladder"].append(run("base: per-token retrieval, per-head selection, four-call kernels",
                              BASE.replace(tau=2.0, k_planted=BASE.k_planted), per_head=True, fused=False))
    rows["ladder"].append(run("+SR: semantic-boundary trigger tau=0.7", BASE, per_head=True, fused=False))
    rows["ladder"].append(run("+GS: group-consistent selection", BASE, per_head=False, fused=False))
    rows["ladder"].append(run("+CK: single-launch retrieval kernel (LouisKV)", BASE, per_head=False, fused=True))
    base_ms = rows["ladder"][0]["ms_per_step"]
    for i, r in enumerate(rows["ladder"]):
        r["speedup_vs_base"] = base_ms / r["ms_per_step"]
        if i:
            r["gain_vs_previous"] = rows["ladder"][i - 1]["ms_per_step"] / r["ms_per_step"] - 1
if args.only in ("", "tau"):
    for tau in (0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.85, 0.9, 0.95):
        rows["tau_sweep"].append(run(f"tau={tau} (graded drift)", BASE.replace(tau=tau, drift=2.0,
                                                                               k_planted=BASE.k_planted)))
if args.only in ("", "policies"):
    rows["policies"].append(run("fixed stride 5", BASE, stride=5))
    rows["policies"].append(run("fixed stride 16", BASE, stride=16))
    rows["policies"].append(run("pages of 16, tau=0.7", BASE, units="pages"))
if args.only == "fetch":
    C2T = C2.replace(k_planted=max(C2.n_clusters // 4, 16))
    rows["fetch"] = [run("C2 zero-copy gather, four calls, eager", C2T, fused=False, graph=False),
                     run("C2 batched DMA gather, four calls, eager", C2T, fused=False, graph=False,
                         fetch=lkv.FETCH_BATCHED_DMA),
                     run("C2 zero-copy gather, single launch, graph (the bench's mode)", C2T)]
    for r in rows["fetch"]:
        r["h2d_GBps_over_step"] = r["h2d_MB_per_step"] / r["ms_per_step"]
if args.only == "index":
    C2T = C2.replace(k_planted=max(C2.n_clusters // 4, 16))
    rows["index"] = [run("C2 index on the device", C2T), run("C2 index in host DRAM", C2T, index_offload=1),
                     run("C4 shape 32K batch 2, index on the device", BASE),
                     run("C4 shape 32K batch 2, index in host DRAM", BASE, index_offload=1)]
if args.only == "fp8":
    C2T = C2.replace(k_planted=max(C2.n_clusters // 4, 16))
    rows["fp8"] = [run("C2 bf16 pool", C2T), run("C2 E4M3 pool", C2T, pool_dtype=lkv.POOL_FP8_E4M3),
                   run("C4 shape 32K batch 2, bf16 pool", BASE),
                   run("C4 shape 32K batch 2, E4M3 pool", BASE, pool_dtype=lkv.POOL_FP8_E4M3)]
print(json.dumps({"workload": f"Qwen3-8B LILO shape, {args.prompt}-token prompt, batch {args.batch}, "
                              f"S=64 W=256 B=1024 c=16, {args.steps} timed decode steps (synthetic, seed 0)",
                  "paper": "P:189 (SR ~2.6x, GS +13.1%, CK +15.7% on A6000, Qwen3-8B 32K+16K), P:465 (tau)",
                  **rows}, indent=1))
