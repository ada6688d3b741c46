"""Probe: graph-replayed C2 decode-step latency under forced trigger regimes.

tau=-2 never flags after t=1 (latency chain only), tau=2 flags every step (selection + host
gather every layer), default tau = the workload's. `--unfused` uses append_output + sparse_attn
for the retrieval layers instead of the clustered append_attn kernel.
"""
import argparse, json, sys, time
import torch
sys.path.insert(0, '.')
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--taus", default="-2,2,default")
ap.add_argument("--unfused", action="store_true")
ap.add_argument("--layer", action="store_true", help="louiskv_decode_layer per layer")
ap.add_argument("--attn-impl", type=int, default=0, help="full-cache attention: 0 tensor cores, 1 SIMT")
args = ap.parse_args()
base = CONFIGS[args.config]
dev = torch.device("cuda", 0)
res = {}
for tau_s in args.taus.split(","):
    cfg = base if tau_s == "default" else base.replace(tau=float(tau_s))
    L, full = cfg.num_layers, set(cfg.full_cache_layers)
    T = 2 + 8 + 2 * args.steps
    ctx = lkv.Context(lkv.make_config(cfg, max_output_len=T + 1, attn_impl=args.attn_impl))
    plants = [synth.planted(cfg, l, 0, dev) for l in range(L)]
    for l in range(L):
        K, V = synth.prompt_kv(cfg, l, 0, dev, plants[l])
        ctx.cluster_prompt(l, K, V)
        del K, V
    q, kk, vv, _ = synth.decode_stream(cfg, T, 0, dev, plants)
    del plants
    q_in, k_in, v_in = q[0].clone(), kk[0].clone(), vv[0].clone()
    out = torch.empty_like(q_in)

    def issue():
        for l in range(L):
            if args.layer:
                ctx.decode_layer(l, q_in[l], k_in[l], v_in[l], out[l])
                continue
            ctx.should_retrieve(l, q_in[l])
            ctx.retrieve(l, q_in[l])
            if l in full or args.unfused:
                ctx.append_output(l, k_in[l], v_in[l])
                ctx.sparse_attn(l, q_in[l], out[l])
            else:
                ctx.append_attn(l, k_in[l], v_in[l], q_in[l], out[l])

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
    rl = (L - len(full)) * cfg.batch * cfg.num_kv_heads
    res[tau_s] = {"ms_per_step": ms,
                  "flag_frac": (st1["retrievals"] - st0["retrievals"]) / (args.steps * (L - len(full)) * cfg.batch),
                  "h2d_MB_per_step": (st1["bytes_h2d"] - st0["bytes_h2d"]) / args.steps / 1e6}
    print(tau_s, json.dumps(res[tau_s]), flush=True)
    del ctx, g
    torch.cuda.empty_cache()
print(json.dumps(res))
