"""Probe: per-phase timeline of the retrieval-layer kernel inside the graph-replayed C2 step.

Needs the profiling build (python paper_2510_11292_b200/build.py --prof); loads it through
LOUISKV_LIB. Slots (globaltimer ns, thread 0 of every CTA): 0 entry, 1 after griddepcontrol.wait,
2 state read, 3 trigger done, 4 select done (flagged), 5 gather done, 6 append done (rank 0),
7 after publish barrier, 8 first attention chunk landed, 9 main loop done, 10/11 merge barrier,
12/13 final barrier, 14 exit; 24 after the L2 prefetch, 25 speculative attention loads issued,
26 trigger math done (before the block barrier), 27 tid 0 flag + window done. Reports medians relative to the launch's earliest entry.
"""
import ctypes, json, os, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
os.environ["LOUISKV_LIB"] = os.path.join(ROOT, "paper_2510_11292_b200", "liblouiskv_prof.so")
sys.path.insert(0, ROOT)
import torch
import paper_2510_11292_b200 as lkv
import synth
from synth.configs import CONFIGS

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tau = float(sys.argv[2]) if len(sys.argv) > 2 else None
if tau is not None:
    cfg = cfg.replace(tau=tau)
if os.environ.get("LKV_PROBE_BATCH"):  # (e.g. C5's per-GPU share: batch 16, one KV head)
    cfg = cfg.replace(batch=int(os.environ["LKV_PROBE_BATCH"]), k_planted=max(cfg.n_clusters // 4, 16))
dev = torch.device("cuda", 0)
L, full, b = cfg.num_layers, set(cfg.full_cache_layers), cfg.batch
Hkv = int(os.environ.get("LKV_PROBE_HEADS", cfg.num_kv_heads))  # owned KV heads [0, Hkv)
STEPS = 24
ctx = lkv.Context(lkv.make_config(cfg, max_output_len=STEPS + 4, kv_head_count=Hkv))
plants = [synth.planted(cfg, l, 0, dev) for l in range(L)]
for l in range(L):
    K, V = synth.prompt_kv(cfg, l, 0, dev, plants[l])
    ctx.cluster_prompt(l, K[:, :, :Hkv], V[:, :, :Hkv])
    del K, V
q, kk, vv, _ = synth.decode_stream(cfg, STEPS + 2, 0, dev, plants)
q_in, k_in, v_in = q[0].clone(), kk[0].clone(), vv[0].clone()
out = torch.empty((L, b, cfg.group * Hkv, cfg.head_dim), dtype=q_in.dtype, device=dev)
flags = torch.zeros((L, b), dtype=torch.uint8, device=dev)


def issue():
    for l in range(L):
        ctx.decode_layer(l, q_in[l], k_in[l][:, :Hkv], v_in[l][:, :Hkv], out[l], flag_out=flags[l])


issue()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.graph(g, stream=s):
    issue()
rd = lkv.lib().louiskv_prof_read
rd.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
clr = lkv.lib().louiskv_prof_clear
ORDER = [0, 1, 2, 24, 25, 26, 27, 3, 20, 6, 13, 16, 17, 15, 18, 19, 4, 5, 7, 8, 9, 10, 11, 12, 14]
deltas = {"unflagged": [], "flagged": []}
buf = np.zeros((64, 2048, 32), np.uint64)
CL = int(os.environ.get("LOUISKV_LAYER_CL", "0")) or (8 if b * Hkv * 8 <= 148 else 4 if b * Hkv * 4 <= 148 else 2)
n_cta = b * Hkv * CL
rows = {"unflagged": [], "flagged": []}
gaps = []
for i in range(1, STEPS + 1):
    q_in.copy_(q[i]); k_in.copy_(kk[i]); v_in.copy_(vv[i])
    torch.cuda.synchronize()
    clr()
    g.replay()
    torch.cuda.synchronize()
    if i < 4:
        continue
    assert rd(buf.ctypes.data, buf.nbytes) == 0
    fl = flags.cpu().numpy()
    prev_end = None
    for l in range(L):
        if l in full:
            prev_end = None
            continue
        t = buf[l, :n_cta].astype(np.int64)
        t0 = t[:, 0].min()
        rel = (t - t0).astype(np.float64)
        rel[t == 0] = np.nan
        rel[:, 21] = t[:, 21]  # a count, not a time
        ok = (t[:, 23] > t[:, 22]) & (t[:, 4] > t[:, 3])
        rel[:, 22] = np.where(ok, (t[:, 23] - t[:, 22]) / np.maximum(t[:, 4] - t[:, 3], 1), np.nan)  # SM GHz
        rel[:, 23] = np.nan
        # per CTA: time from the previous present stamp (program order), median over the CTAs of the
        # flagged (resp. unflagged) instances of this launch
        cta_flag = np.array([fl[l][(c // CL) // Hkv] for c in range(n_cta)], bool)
        for key, sel in (("flagged", cta_flag), ("unflagged", ~cta_flag)):
          if not sel.any():
            continue
          dl = {}
          for c in np.nonzero(sel)[0]:
            prev = None
            for sl in ORDER:
                if t[c, sl] == 0:
                    continue
                if prev is not None:
                    dl.setdefault(f"{prev}->{sl}", []).append(int(t[c, sl] - t[c, prev]))
                prev = sl
          deltas[key].append({k_: float(np.median(v_)) for k_, v_ in dl.items()})
          rows[key].append(np.nanmedian(rel[sel], axis=0).tolist() + [np.nanmax(rel[sel][:, 14])])
        buf[l] = 0
        if prev_end is not None:
            gaps.append(t0 - prev_end)
        prev_end = t[:, 14].max()
res = {k: (np.median(np.array(v), axis=0).round(0).tolist() if v else None) for k, v in rows.items()}
res["n"] = {k: len(v) for k, v in rows.items()}
res["gap_prev_exit_to_entry_ns_median"] = float(np.median(gaps)) if gaps else None
for k_, lst in deltas.items():
    if lst:
        keys = sorted({x for d_ in lst for x in d_}, key=lambda z: ORDER.index(int(z.split("->")[1])))
        res["delta_" + k_] = {x: float(np.median([d_[x] for d_ in lst if x in d_])) for x in keys}
print(json.dumps(res))
