"""Tiny runs of every kernel for compute-sanitizer (memcheck / racecheck / synccheck):
prompt clustering (tcgen05 + SIMT assignment, page units, caller-supplied units), the four per-step ABI
calls, the fused append+attention, the single-launch layer kernel at cluster sizes 8 and 2 (incl. the
big-mode select with > 8192 live units), full-cache layers (tensor-core and SIMT attention), (r2) the
BATCHED_DMA fetch, the host-resident index and the E4M3 pool.
usage: compute-sanitizer --tool <tool> python tools/sanitize.py"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))
import numpy as np
import torch

import paper_2510_11292_b200 as lkv
from synth.configs import Config
from _pair import make_inputs, planted_assign

base = Config("san", num_layers=2, num_q_heads=8, num_kv_heads=2, head_dim=128, batch=1, prompt_len=700,
              decode_steps=6, sink_tokens=8, window_tokens=16, budget_tokens=64, tau=0.85, avg_cluster_size=16,
              kmeans_iters=2, full_cache_layers=(0,), seg_mean=3.0)


def episode(cfg, steps, mode, units=lkv.UNITS_KMEANS, kimpl=0, aimpl=0, assign=None, **variant):
    inp = make_inputs(cfg, steps, 1)
    ctx = lkv.Context(lkv.make_config(cfg, kmeans_impl=kimpl, attn_impl=aimpl, prompt_units=units, **variant))
    for l in range(cfg.num_layers):
        if assign is not None and l not in cfg.full_cache_layers:
            a = assign(cfg, inp, l)
            k = int(a.max()) + 1
            cen = np.zeros((cfg.batch, cfg.num_kv_heads, k, 128), np.float32)
            ctx.set_prompt_units(l, inp.K[l], inp.V[l], a, cen)
        else:
            ctx.cluster_prompt(l, inp.K[l], inp.V[l])
    ctx.prompt_fence()
    b, g, hn = cfg.batch, cfg.group, cfg.num_kv_heads
    out = torch.zeros((b, g * hn, 128), dtype=torch.bfloat16, device="cuda")
    o32 = torch.zeros((b, g * hn, 128), dtype=torch.float32, device="cuda")
    for t in range(steps):
        for l in range(cfg.num_layers):
            q, k, v = inp.q[t, l], inp.k[t, l].contiguous(), inp.v[t, l].contiguous()
            if mode == "layer":
                ctx.decode_layer(l, q, k, v, out, o32)
            elif mode == "fused":
                ctx.should_retrieve(l, q)
                ctx.retrieve(l, q)
                ctx.append_attn(l, k, v, q, out, o32)
            else:
                ctx.should_retrieve(l, q)
                ctx.retrieve(l, q)
                ctx.append_output(l, k, v)
                ctx.sparse_attn(l, q, out, o32)
    torch.cuda.synchronize()
    st = ctx.stats()
    ctx.close()
    return st


runs = [
    ("four-call, tcgen05 k-means", lambda: episode(base, 6, "calls")),
    ("append_attn, SIMT k-means, SIMT full attention", lambda: episode(base, 6, "fused", kimpl=1, aimpl=1)),
    ("decode_layer CL=8", lambda: episode(base, 6, "layer")),
    ("decode_layer pages", lambda: episode(base, 4, "layer", units=lkv.UNITS_PAGES)),
    ("four-call, BATCHED_DMA fetch", lambda: episode(base, 6, "calls", fetch_mode=lkv.FETCH_BATCHED_DMA)),
    ("decode_layer, index offload", lambda: episode(base, 6, "layer", index_offload=1)),
    ("four-call, index offload", lambda: episode(base, 6, "calls", index_offload=1)),
    ("decode_layer, E4M3 pool", lambda: episode(base, 6, "layer", pool_dtype=lkv.POOL_FP8_E4M3)),
    ("append_attn, E4M3 pool", lambda: episode(base, 6, "fused", pool_dtype=lkv.POOL_FP8_E4M3)),
]


def many(cfg, inp, l):
    N = cfg.prompt_len - cfg.sink_tokens
    return np.arange(N, dtype=np.int32)[None, None, :].repeat(cfg.num_kv_heads, 1)


big = base.replace(num_layers=1, full_cache_layers=(), num_kv_heads=1, num_q_heads=4, prompt_len=8300,
                   avg_cluster_size=1, budget_tokens=128, tau=2.0)
runs.append(("decode_layer big-mode select (8292 units)", lambda: episode(big, 2, "layer", assign=many)))
for name, fn in runs:
    st = fn()
    print(f"OK {name}: retrievals {st['retrievals']}, fetched {st['units_fetched']}", flush=True)
os.environ["LOUISKV_LAYER_CL"] = "2"
st = episode(base.replace(batch=2), 6, "layer")
print(f"OK decode_layer CL=2: retrievals {st['retrievals']}", flush=True)
print("sanitize runs complete")
