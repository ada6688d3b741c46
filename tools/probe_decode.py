"""Probe: a few graph-free decode steps of the C2 workload (all 32 layers) for ncu."""
import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import C2
cfg = C2
T = 12
ctx = lkv.Context(lkv.make_config(cfg, kmeans_impl=0))
plants = [synth.planted(cfg, l, 0, "cuda") for l in range(cfg.num_layers)]
for l in range(cfg.num_layers):
    K, V = synth.prompt_kv(cfg, l, 0, "cuda", plants[l])
    ctx.cluster_prompt(l, K, V)
q, k, v, _ = synth.decode_stream(cfg, T, 0, "cuda", plants)
out = torch.empty((cfg.num_layers, 1, 32, 128), dtype=torch.bfloat16, device="cuda")
for t in range(T):
    for l in range(cfg.num_layers):
        ctx.should_retrieve(l, q[t, l]); ctx.retrieve(l, q[t, l]); ctx.append_attn(l, k[t, l], v[t, l], q[t, l], out[l])
torch.cuda.synchronize()
print(ctx.stats())
