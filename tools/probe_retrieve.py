"""Probe: time retrieve (score_select + gather) on one C2 retrieval layer, retrieval forced
every step (tau > 1). Run under ncu to split the kernels."""
import os, sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2510_11292_b200 as lkv
from synth.configs import C1, C2
from _pair import make_inputs
inp = make_inputs(C1, 1, 0, layout="blocked")
ctx = lkv.Context(lkv.make_config(C1))
ctx.cluster_prompt(0, inp.K[0], inp.V[0])
print("C1 kmeans stats", ctx.stats())
ctx.close()
cfg = C2.replace(num_layers=1, full_cache_layers=(), tau=float(os.environ.get("TAU", "1.01")), decode_steps=24)
inp = make_inputs(cfg, 24, 0)
ctx = lkv.Context(lkv.make_config(cfg))
ctx.cluster_prompt(0, inp.K[0], inp.V[0])
out = torch.empty((1, 32, 128), dtype=torch.bfloat16, device="cuda")
ts = []
for t in range(24):
    ctx.should_retrieve(0, inp.q[t, 0])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.retrieve(0, inp.q[t, 0])
    e1.record()
    ctx.append_output(0, inp.k[t, 0], inp.v[t, 0])
    ctx.sparse_attn(0, inp.q[t, 0], out)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("retrieve ms per call:", [round(x, 3) for x in ts])
print(ctx.stats())
