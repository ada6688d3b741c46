"""Probe: per-phase device time of cluster_prompt (library prefill timer) on C2 / C4 layers, per
layer-iteration, for A/B of the k-means kernels (LOUISKV_LIB selects a variant build).
usage: python tools/probe_kmeans_phases.py [C2|C4] [layers]"""
import json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
cfg = cfg.replace(num_layers=nl + 1, full_cache_layers=(), k_planted=max(cfg.n_clusters // 4, 16))
ctx = lkv.Context(lkv.make_config(cfg, max_output_len=8))
K, V = synth.prompt_kv(cfg, 0, 0, "cuda")
ctx.cluster_prompt(0, K, V)  # warm-up layer
torch.cuda.synchronize()
ctx.set_prefill_timing(True)
for l in range(1, nl + 1):
    ctx.cluster_prompt(l, K, V)
ctx.prompt_fence()
torch.cuda.synchronize()
t = ctx.prefill_times()
it = t["assign_passes"]
out = {k: t[k] / it * 1e3 for k in ("assign_ms", "sort_ms", "update_ms")}
out = {"config": name, "lib": os.path.basename(lkv.LIB_PATH), "us_per_layer_iteration": out,
       "non_gemm_share": (out["sort_ms"] + out["update_ms"]) / sum(out.values()), "passes": it}
print(json.dumps(out))
