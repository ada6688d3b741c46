"""Prompt clustering overlapped with a stand-in prefill forward (the paper's
"asynchronously with the prefill forward pass, avoiding blocking").

C2 shape (Llama-3.1-8B: 32 layers, d_model 4096, 32 query / 8 KV heads, MLP 14336), 32K-token prompt.
The stand-in prefill of one layer is its weight GEMMs at that shape with random bf16 weights
(QKV 4096x6144, O 4096x4096, gate+up 4096x28672, down 14336x4096 — cuBLAS, as a model would run
them; the attention itself is left out). louiskv_cluster_prompt of layer l (k-means + the
cluster-major offload to the pinned pool) is issued on a side stream after layer l's GEMMs, so it
runs concurrently with layer l+1's. Reported: prefill alone, clustering alone, both overlapped
(device time, CUDA events), and the clustering time the overlap hides.
usage: python tools/prefill_overlap.py [--layers 32]
"""
import argparse, json, os, sys
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import torch
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=32)
args = ap.parse_args()
cfg = CONFIGS["C2"].replace(num_layers=args.layers)
dev = torch.device("cuda", 0)
L, P, dm = cfg.num_layers, cfg.prompt_len, 4096
g = torch.Generator(device=dev).manual_seed(0)
W = [torch.randn(dm, n, device=dev, dtype=torch.bfloat16, generator=g) * 0.02 for n in (6144, 4096, 28672)]
Wd = torch.randn(14336, dm, device=dev, dtype=torch.bfloat16, generator=g) * 0.02
x = torch.randn(P, dm, device=dev, dtype=torch.bfloat16, generator=g)
plants = [synth.planted(cfg, l, 0, dev) for l in range(L)]
prompts = [synth.prompt_kv(cfg, l, 0, dev, plants[l]) for l in range(L)]
main, side = torch.cuda.current_stream(), torch.cuda.Stream()


def layer_gemms():
    qkv = x @ W[0]
    o = x @ W[1]
    gu = x @ W[2]
    h = torch.nn.functional.silu(gu[:, :14336]) * gu[:, 14336:]
    return (h @ Wd).add_(o).sum() + qkv[0, 0]


def run(prefill: bool, cluster: bool):
    ctx = lkv.Context(lkv.make_config(cfg, max_output_len=8)) if cluster else None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for l in range(L):
        if prefill:
            layer_gemms()
        if cluster:
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)  # layer l's K, V exist once its GEMMs are issued before
            with torch.cuda.stream(side):
                ctx.cluster_prompt(l, *prompts[l], stream=side)
    if cluster:
        with torch.cuda.stream(side):
            ctx.prompt_fence(stream=side)
        ev = torch.cuda.Event()
        ev.record(side)
        main.wait_event(ev)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if ctx is not None:
        ctx.close()
    return ms


run(True, True)  # warm-up (cuBLAS heuristics, kernel attributes)
t_p = run(True, False)
t_c = run(False, True)
t_b = run(True, True)
print(json.dumps({"config": cfg.name, "layers": L, "prompt_len": P,
                  "prefill_gemms_ms": t_p, "cluster_prompt_ms": t_c, "overlapped_ms": t_b,
                  "hidden_frac_of_clustering": max(0.0, (t_p + t_c - t_b) / t_c) if t_c > 0 else None,
                  "slowdown_of_prefill": t_b / t_p - 1.0,
                  "note": "stand-in prefill = the layer's weight GEMMs (cuBLAS, random bf16 weights); clustering on a "
                          "side stream after each layer's GEMMs; device time by CUDA events"}, indent=1))
