"""Probe: cluster_prompt on C2 layers (tcgen05 path) for an ncu launch list."""
import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import C2
cfg = C2.replace(num_layers=2, full_cache_layers=())
ctx = lkv.Context(lkv.make_config(cfg))
for l in range(2):
    K, V = synth.prompt_kv(cfg, l, 0, "cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.cluster_prompt(l, K, V); e1.record(); torch.cuda.synchronize()
    print("layer", l, "cluster_prompt ms", e0.elapsed_time(e1))
print(ctx.stats())
