"""Probe: device time of the full-cache decode attention (layers 0-1 of C2) alone, graph-replayed.

usage: python tools/probe_full.py [attn_impl] [reps]  (attn_impl 0 = tensor cores (default), 1 = SIMT)
Environment variables read by the library select load-path experiments (LOUISKV_FA_TMA)."""
import json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

impl = int(sys.argv[1]) if len(sys.argv) > 1 else 0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = CONFIGS[os.environ.get("LKV_PROBE_CFG", "C2")]  # (env: another config, batch, owned KV heads)
if os.environ.get("LKV_PROBE_BATCH"):
    cfg = cfg.replace(batch=int(os.environ["LKV_PROBE_BATCH"]))
hc = int(os.environ.get("LKV_PROBE_HEADS", cfg.num_kv_heads))
if len(sys.argv) > 3:
    cfg = cfg.replace(prompt_len=int(sys.argv[3]))
dev = torch.device("cuda", 0)
ctx = lkv.Context(lkv.make_config(cfg, max_output_len=2 * reps + 64, attn_impl=impl, kv_head_count=hc))
layers = sorted(cfg.full_cache_layers)
plants = {l: synth.planted(cfg, l, 0, dev) for l in layers}
for l in layers:
    Kp, Vp = synth.prompt_kv(cfg, l, 0, dev, plants[l])
    ctx.cluster_prompt(l, Kp[:, :, :hc], Vp[:, :, :hc])
    del Kp, Vp
torch.cuda.synchronize()
q = torch.randn((cfg.num_layers, cfg.batch, cfg.num_q_heads, cfg.head_dim), device=dev).bfloat16()
k = torch.randn((cfg.num_layers, cfg.batch, hc, cfg.head_dim), device=dev).bfloat16()
out = torch.empty((cfg.num_layers, cfg.batch, cfg.group * hc, cfg.head_dim), device=dev).bfloat16()
for l in layers:
    ctx.decode_layer(l, q[l], k[l], k[l], out[l])
torch.cuda.synchronize()
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    for l in layers:
        ctx.decode_layer(l, q[l], k[l], k[l], out[l])
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(reps // 2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) / len(layers))
ts.sort()
# back to back (no host sync between replays): the device stays busy, as inside a decode step
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps // 2):
    g.replay()
b.record()
torch.cuda.synchronize()
b2b = a.elapsed_time(b) / (reps // 2) / len(layers)
rows = cfg.prompt_len + reps
byts = cfg.batch * hc * rows * 512
med = ts[len(ts) // 2]
print(json.dumps({"P": cfg.prompt_len, "impl": impl, "tma": bool(os.environ.get("LOUISKV_FA_TMA")), "us_per_layer_median": med * 1e3,
                  "us_min": ts[0] * 1e3, "us_back_to_back": b2b * 1e3, "GBps_b2b": byts / (b2b / 1e3) / 1e9, "GBps": byts / (med / 1e3) / 1e9, "bytes": byts}))
ctx.close()

if len(sys.argv) > 4:  # plain torch read of the same byte count, for comparison
    x = torch.empty(byts // 2, dtype=torch.bfloat16, device=dev).normal_()
    y = torch.empty(1, dtype=torch.float32, device=dev)
    for _ in range(3):
        y = x.sum(dtype=torch.float32)
    ts = []
    for _ in range(50):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); y = x.sum(dtype=torch.float32); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        y = x.sum(dtype=torch.float32)
    b.record(); torch.cuda.synchronize()
    t2 = a.elapsed_time(b) / 50
    print(json.dumps({"torch_sum_us": ts[25] * 1e3, "GBps": byts / (ts[25] / 1e3) / 1e9, "b2b_us": t2 * 1e3,
                      "GBps_b2b": byts / (t2 / 1e3) / 1e9}))
