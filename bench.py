#!/usr/bin/env python
"""LouisKV retrieval hot path on B200 — benchmark (driver contract: one JSON line).

Workload (BASELINE.json configs[1]): Llama-3.1-8B attention shape
(32 layers, 32 query heads, 8 KV heads GQA, d=128), 32K-token prompt, batch 1,
S=32 / W=512 / B=512 / tau=0.85 / c=16, first two layers full-cache.
Synthetic seeded data (synth/), random-init: there are no weights in this path.

One timed "step" = one decode step through all 32 layers in model order, each layer:
should_retrieve -> retrieve (score/select/gather on flagged sequences) -> append_output
-> sparse_attn (full-cache layers: dense attention), replayed as one CUDA graph with inputs
already resident in HBM. The prompt clustering (cluster_prompt, once per layer) is timed
separately and reported as k-means keys/s. Multi-GPU (torchrun): weak scaling, every rank
runs its own independent sequence batch (no data-path collective; SURVEY §8(e) partitioning
by batch). ``--impl reference`` times the CPU oracle (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "decode tok/s with LouisKV retrieval at 32K ctx; k-means keys/s; retrieve µs/step"
UNIT = "tok/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=256)
    p.add_argument("--warmup", type=int, default=16)
    p.add_argument("--impl", default="product", choices=["product", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--attr-steps", type=int, default=64, help="steps of the per-phase attribution pass")
    p.add_argument("--cpu-steps", type=int, default=48, help="oracle decode steps for cpu_baseline")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--kmeans-impl", type=int, default=0)
    p.add_argument("--shard", default="batch", choices=["batch", "heads"],
                   help="multi-GPU partitioning: 'batch' = every rank its own sequences (weak scaling, no "
                        "collective); 'heads' = ranks own contiguous KV-head ranges of the same sequences and "
                        "all-gather the per-head attention outputs over NCCL after every layer (strong scaling)")
    return p.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device_index: int):
        self.idx = device_index
        self.proc = None
        self.out = None

    def start(self):
        try:
            self.out = open(os.path.join("/tmp", f"lkv_clocks_{os.getpid()}.csv"), "w+")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.seek(0)
        rows = [l.strip().split(",") for l in self.out.read().splitlines() if l.strip()]
        self.out.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[3:7]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(n)
            except Exception:
                continue
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def rank_seed(seed: int, rank: int) -> int:
    """Weak scaling: every rank draws its own independent sequences."""
    return seed + 1000 * rank


def head_range(rank: int, world: int, num_kv_heads: int):
    """KV-head shard of `rank`: contiguous ranges, num_kv_heads / world heads each."""
    if num_kv_heads % world:
        raise ValueError(f"--shard heads needs num_kv_heads ({num_kv_heads}) divisible by the world size ({world})")
    hc = num_kv_heads // world
    return rank * hc, hc


def gather_heads(out_own, gathered, world: int):
    """All-gather of one layer's per-head attention outputs (north_star: NCCL over NVLink, only for the
    outputs). out_own [b, g*hc, d] -> gathered [world, b, g*hc, d] (rank-major: rank r holds query heads
    [r*g*hc, (r+1)*g*hc)). Stream-ordered, so it is captured into the step's CUDA graph."""
    if world > 1:
        import torch.distributed as dist
        dist.all_gather_into_tensor(gathered.view((-1,) + tuple(out_own.shape[1:])), out_own)
    else:
        gathered[0].copy_(out_own)


def assemble_heads(gathered):
    """[world, b, g*hc, d] -> [b, Hq, d] in model head order (what the O-projection consumes)."""
    w, b, gh, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(b, w * gh, d)


def ncu_traffic():
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant kernels from
    the committed `ncu --set full` capture summary (profiles/r01_traffic.json); {} when absent."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "r01_traffic.json")))
    except Exception:
        return {}


def max_over_ranks(x: float, world: int) -> float:
    """Max of a per-rank device time over all ranks (nccl on GPUs, gloo in the CPU tests)."""
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


# ----------------------------------------------------------------------------- oracle (CPU) leg
def oracle_sample(cfg, seed: int, steps: int):
    """Time the CPU oracle, as it stands, on a bounded sample of the workload: one retrieval-layer
    instance (1 KV head, its g query heads) and one full-cache instance of the C2 shape, `steps`
    decode steps. Returns per-instance-step seconds and the extrapolated full decode-step time
    (inst counts of the config: b*L_r*Hkv retrieval + b*L_f*Hkv full-cache instances)."""
    import numpy as np
    import torch
    import synth
    from oracle.episode import OracleEpisode
    from _pair import planted_assign

    one = cfg.replace(num_layers=2, full_cache_layers=(0,), num_kv_heads=1, num_q_heads=cfg.group, batch=1,
                      decode_steps=steps, k_planted=cfg.k_planted)
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    plants = [synth.planted(one, l, seed, dev) for l in range(2)]
    KV = [synth.prompt_kv(one, l, seed, dev, plants[l], return_labels=True) for l in range(2)]
    q, k, v, _ = synth.decode_stream(one, steps, seed, dev, plants)
    ep = OracleEpisode(one)
    ep.cluster_prompt(0, KV[0][0].float().cpu().numpy(), KV[0][1].float().cpu().numpy())
    a = planted_assign(one, KV[1][2])
    ep.cluster_prompt(1, KV[1][0].float().cpu().numpy(), KV[1][1].float().cpu().numpy(), assign=a)
    qn, kn, vn = q.float().cpu().numpy(), k.float().cpu().numpy(), v.float().cpu().numpy()
    t_full = t_ret = 0.0
    for t in range(steps):
        for l in range(2):
            t0 = time.perf_counter()
            ep.should_retrieve(l, qn[t, l])
            ep.retrieve(l, qn[t, l])
            ep.append_output(l, kn[t, l], vn[t, l])
            ep.sparse_attn(l, qn[t, l])
            dt = time.perf_counter() - t0
            if l == 0:
                t_full += dt
            else:
                t_ret += dt
    n_full = cfg.batch * len(cfg.full_cache_layers) * cfg.num_kv_heads
    n_ret = cfg.batch * (cfg.num_layers - len(cfg.full_cache_layers)) * cfg.num_kv_heads
    step_s = (n_ret * t_ret + n_full * t_full) / steps
    return dict(t_ret=t_ret / steps, t_full=t_full / steps, step_s=step_s, n_ret=n_ret, n_full=n_full)


def run_reference(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from synth.configs import CONFIGS
    cfg = CONFIGS[args.config]
    total = args.warmup + args.steps
    s = oracle_sample(cfg, args.seed, total)
    value = cfg.batch / s["step_s"]
    sample = (f"per step: 1 retrieval-layer instance (1 KV head, {cfg.group} q heads) + 1 full-cache instance of "
              f"{cfg.name}, extrapolated x{s['n_ret']} / x{s['n_full']} instances; {total} steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": s["step_s"] * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"{cfg.name}", "global_batch": cfg.batch * args.gpus,
                                            "seq_len": cfg.prompt_len},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- product leg
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import synth
    from synth.configs import CONFIGS
    import paper_2510_11292_b200 as lkv

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    L, b, Hq, Hkv, d, g = cfg.num_layers, cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.group
    full = set(cfg.full_cache_layers)
    K, W = args.steps, args.warmup
    A = args.attr_steps
    T = 1 + W + K + K + A + 2  # direct step + warmup + timed + e2e + attribution (+slack)
    heads = args.shard == "heads"
    # batch sharding: every rank its own sequences; head sharding: the same sequences, own KV heads
    seed = args.seed if heads else rank_seed(args.seed, rank)
    hb, hc = head_range(rank, world, Hkv) if heads else (0, Hkv)
    gq = g * hc  # query heads owned by this rank
    jobs = 1 if heads else world  # independent sequence batches processed by the whole job
    ctx = lkv.Context(lkv.make_config(cfg, kv_head_begin=hb, kv_head_count=hc,
                                      max_output_len=max(cfg.max_output_len, T + 1), device=local,
                                      kmeans_impl=args.kmeans_impl))

    # ---------------- prefill: cluster_prompt for every layer, timed as one region ending at the
    # prompt fence (k-means keys/s; the copy-engine offload of layer l overlaps layer l+1's k-means)
    plants = [synth.planted(cfg, l, seed, dev) for l in range(L)]
    prompts = [tuple(t[:, :, hb:hb + hc] for t in synth.prompt_kv(cfg, l, seed, dev, plants[l])) for l in range(L)]
    km_keys = sum(b * hc * (cfg.prompt_len - cfg.sink_tokens) for l in range(L) if l not in full)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for l in range(L):
        ctx.cluster_prompt(l, *prompts[l])
    ctx.prompt_fence()
    e1.record()
    torch.cuda.synchronize()
    km_ms = max_over_ranks(e0.elapsed_time(e1), world)
    km_keys *= world  # keys clustered by the whole job (every rank: its own heads or sequences)
    del prompts
    st0 = ctx.stats()

    # ---------------- decode inputs (device resident) and static graph buffers
    q, kk, vv, bset = synth.decode_stream(cfg, T, seed, dev, plants)
    del plants
    # one step's inputs (q of all heads, k_t, v_t of every layer) packed in ONE buffer, so a step's
    # input is a single copy: qkv [T, n_q + 2 n_kv] on the device (and pinned on the host for e2e)
    n_q, n_kv = L * b * Hq * d, L * b * Hkv * d
    qkv = torch.cat([q.reshape(T, -1), kk.reshape(T, -1), vv.reshape(T, -1)], dim=1)
    del q, kk, vv
    qkv_in = torch.empty((n_q + 2 * n_kv,), dtype=torch.bfloat16, device=dev)
    q_in = qkv_in[:n_q].view(L, b, Hq, d)
    k_in = qkv_in[n_q:n_q + n_kv].view(L, b, Hkv, d)
    v_in = qkv_in[n_q + n_kv:].view(L, b, Hkv, d)
    out = torch.empty((L, b, gq, d), dtype=torch.bfloat16, device=dev)
    # head sharding: per-layer all-gather of the owned heads' outputs -> [L, world, b, gq, d]
    gathered = torch.empty((L, world, b, gq, d), dtype=torch.bfloat16, device=dev) if heads else None
    k_own = k_in[:, :, hb:hb + hc]
    v_own = v_in[:, :, hb:hb + hc]

    flags = torch.zeros((L, b), dtype=torch.uint8, device=dev)

    def issue_step(events=None, src=None):
        # one louiskv_decode_layer call per layer: trigger -> retrieve -> store_cache -> attention
        # (one clustered launch on a retrieval layer; one launch on a full-cache layer). src: a step's
        # packed inputs read in place (else the static input buffer)
        qs, ks, vs = q_in, k_own, v_own
        if src is not None:
            qs = src[:n_q].view(L, b, Hq, d)
            ks = src[n_q:n_q + n_kv].view(L, b, Hkv, d)[:, :, hb:hb + hc]
            vs = src[n_q + n_kv:].view(L, b, Hkv, d)[:, :, hb:hb + hc]
        for l in range(L):
            if events is not None:
                events[l].record()
            ctx.decode_layer(l, qs[l], ks[l], vs[l], out[l], flag_out=flags[l])
            if heads:
                gather_heads(out[l], gathered[l], world)
        if events is not None:
            events[L].record()

    step_idx = 0

    def load(i):
        qkv_in.copy_(qkv[i], non_blocking=True)

    # step 1 runs directly (sets kernel attributes, t == 1 retrieval everywhere)
    load(step_idx)
    issue_step()
    step_idx += 1
    torch.cuda.synchronize()

    cap_stream = torch.cuda.Stream(device=dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cap_stream):
        issue_step()
    # retrieval layer: one clustered launch (layer_kernel); full-cache layer: one launch
    # (attn_full_tc_kernel with store_cache fused)
    launches_per_step = L

    for _ in range(W):
        load(step_idx)
        graph.replay()
        step_idx += 1
    # the timed region replays one graph per step, each reading its step's inputs in place (already
    # resident in HBM: no per-step copy); captured before the clock starts
    step_graphs = []
    for i in range(K):
        gi = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gi, stream=cap_stream):
            issue_step(src=qkv[step_idx + i])
        step_graphs.append(gi)
    torch.cuda.synchronize()

    # ---------------- timed region (device-resident inputs)
    P_, nr_ = cfg.prompt_len, L - len(full)
    kv_step_bytes = (len(full) * b * hc * (P_ + T) + nr_ * b * hc * (cfg.sink_tokens + cfg.budget_tokens
                                                                      + cfg.window_tokens)) * 512
    L2_BYTES = 126 * 2 ** 20
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if kv_step_bytes < 2 * L2_BYTES else None
    clocks = ClockSampler(local)
    barrier(world)
    clocks.start()
    st_a = ctx.stats()
    barrier(world)
    def dev_timed(body):
        """Device time of K calls of body(i). When the rank's per-step KV bytes fit in L2 (head sharding
        over many GPUs), L2 is flushed between steps, outside the timed spans (per-step event pairs)."""
        if flush_buf is None:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for i in range(K):
                body(i)
            t1.record()
            torch.cuda.synchronize()
            return t0.elapsed_time(t1)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for i in range(K):
            flush_buf.add_(1)
            evs[i][0].record()
            body(i)
            evs[i][1].record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(z) for a, z in evs)

    def timed_body(i):
        nonlocal step_idx
        step_graphs[i].replay()
        step_idx += 1

    ms = dev_timed(timed_body)
    barrier(world)
    clk = clocks.stop()
    ms = max_over_ranks(ms, world)
    st_b = ctx.stats()
    value = jobs * b * K / (ms / 1e3)

    # ---------------- e2e: host inputs -> device, graph, outputs -> host, every step
    qkv_h = qkv[step_idx:step_idx + K].cpu().pin_memory()
    res = gathered if heads else out  # the step's result: every query head's output
    oh = torch.empty((K,) + tuple(res.shape), dtype=torch.bfloat16).pin_memory()
    barrier(world)
    def e2e_body(i):
        nonlocal step_idx
        qkv_in.copy_(qkv_h[i], non_blocking=True)
        graph.replay()
        oh[i].copy_(res, non_blocking=True)
        step_idx += 1

    st_e0 = ctx.stats()
    e2e_ms = dev_timed(e2e_body)
    barrier(world)
    st_e1 = ctx.stats()
    e2e_ms = max_over_ranks(e2e_ms, world)
    e2e = {"value": jobs * b * K / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(qkv_h[0].numel()) * 2,
           "d2h_bytes_per_step": int(oh[0].numel()) * 2, "ms_per_step": e2e_ms / K,
           # (the e2e steps are the K decode steps after the timed ones: their retrieval rate differs)
           "retrievals_per_step": (st_e1["retrievals"] - st_e0["retrievals"]) / K / max(L - len(full), 1) / b}

    # ---------------- attribution pass: the retrieval layers and the full-cache layers captured as two
    # separate graphs (layers are independent, so each keeps its own step sequence; PDL edges intact,
    # no event nodes inside), each replay timed on the device; the retrieval-layer time per launch is
    # split into unflagged / flagged by a least-squares fit over replays (flags read back per replay)
    ret_layers = [l for l in range(L) if l not in full]

    def issue_subset(layers):
        for l in layers:
            ctx.decode_layer(l, q_in[l], k_own[l], v_own[l], out[l], flag_out=flags[l])

    g_ret, g_full = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_ret, stream=cap_stream):
        issue_subset(ret_layers)
    with torch.cuda.graph(g_full, stream=cap_stream):
        issue_subset(sorted(full))
    st_c = ctx.stats()
    rows_fit, t_full = [], []
    for i in range(A):
        load(step_idx)
        step_idx += 1
        a0, a1, a2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        a0.record()
        g_ret.replay()
        a1.record()
        g_full.replay()
        a2.record()
        torch.cuda.synchronize()
        nf = int(flags[ret_layers].any(dim=1).sum().item())
        rows_fit.append((len(ret_layers) - nf, nf, a0.elapsed_time(a1)))
        t_full.append(a1.elapsed_time(a2) / max(len(full), 1))
    st_d = ctx.stats()
    X = np.array([[r[0], r[1]] for r in rows_fit], dtype=np.float64)
    y = np.array([r[2] for r in rows_fit], dtype=np.float64)
    n_unf_tot, n_flg_tot = int(X[:, 0].sum()), int(X[:, 1].sum())
    if n_flg_tot and n_unf_tot:
        coef = np.linalg.lstsq(X, y, rcond=None)[0]
    elif n_flg_tot:
        coef = np.array([0.0, y.sum() / n_flg_tot])
    else:
        coef = np.array([y.sum() / max(n_unf_tot, 1), 0.0])
    u_ms, f_ms = float(coef[0]), float(coef[1])
    mean = lambda xs: sum(xs) / len(xs) if xs else 0.0
    t_unf = [u_ms] * n_unf_tot
    t_flg = [f_ms] * n_flg_tot
    phase = {"retrieval_layers_unflagged": u_ms * n_unf_tot / A, "retrieval_layers_flagged": f_ms * n_flg_tot / A,
             "full_cache_layers": mean(t_full) * len(full)}  # ms per step
    layer_us = {"retrieval_unflagged": u_ms * 1e3, "retrieval_flagged": f_ms * 1e3, "full_cache": mean(t_full) * 1e3,
                "n_flagged": n_flg_tot, "n_unflagged": n_unf_tot,
                "method": "per-replay device time of a retrieval-layers-only graph, least squares on flag counts"}

    # ---------------- host-link peak (pinned H2D copy) and HBM / tensor peaks
    hl = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    hd = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    best = 1e9
    for _ in range(4):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        hd.copy_(hl, non_blocking=True)
        a1.record()
        torch.cuda.synchronize()
        best = min(best, a0.elapsed_time(a1))
    host_link_gbs = (256 << 20) / (best / 1e3) / 1e9
    del hl, hd
    peaks = measured_peaks()
    traffic = ncu_traffic()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)

    # ---- per-launch algorithmic bytes. Full-cache launch: K+V rows of P+t tokens. Retrieval-layer
    # launch: the attended rows (sinks + working set + local buffer; buffered = t - evicted tokens),
    # plus on a flagged launch the centroid reads (n_units x 256 B) and the working-set rebuild
    # (rows written 512 B each; host rows cross the link, kept rows are re-read from HBM).
    P = cfg.prompt_len
    t_mid = step_idx - A // 2
    full_bytes = b * hc * (P + t_mid) * 2 * d * 2
    att_rows, n_units = 0, 0
    kc = -(-(P - cfg.sink_tokens) // cfg.avg_cluster_size)
    for l in range(L):
        if l in full:
            continue
        for bb in range(b):
            for hh in range(hc):
                _, sizes, _ = ctx.get_units(l, bb, hh)
                nws = len(ctx.get_working_set(l, bb, hh)[0])
                att_rows += min(cfg.sink_tokens, P) + nws + (step_idx - int(sizes[kc:].sum()))
                n_units += len(sizes)
    n_rl = L - len(full)
    unf_bytes = att_rows / n_rl * 512
    h2d_bytes = st_d["bytes_h2d"] - st_c["bytes_h2d"]
    flg_launches = max(len(t_flg), 1)
    ws_rows_flg = b * hc * cfg.budget_tokens  # rows rebuilt per flagged launch (upper bound: B per instance)
    flg_bytes = unf_bytes + n_units / n_rl * 256 + ws_rows_flg * 512 + (ws_rows_flg * 512 - h2d_bytes / flg_launches)
    ret_ms = (sum(t_unf) + sum(t_flg)) / max(len(t_unf) + len(t_flg), 1)
    ret_bytes = (unf_bytes * len(t_unf) + flg_bytes * len(t_flg)) / max(len(t_unf) + len(t_flg), 1)
    ret_gbs = ret_bytes / (ret_ms / 1e3) / 1e9
    step_ms_attr = sum(phase.values())
    lk_tr, fa_tr = traffic.get("layer_kernel"), traffic.get("attn_full_tc_kernel")
    n_l = max(len(t_unf) + len(t_flg), 1)
    layer_traffic = ((lk_tr["unflagged"] * len(t_unf) + lk_tr["flagged"] * len(t_flg)) / n_l) if lk_tr else None
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if peaks else "fallback 6650 GB/s"
    roofline_layer = {"kernel": "layer_kernel (retrieval layers: trigger + score/select + gather + append + attention)",
                      "bound": "hbm", "achieved": ret_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": ret_gbs / hbm_peak,
                      "traffic": layer_traffic, "bytes_per_launch": ret_bytes, "ms_per_launch": ret_ms,
                      "peak_source": peak_src,
                      "share_of_step": (phase["retrieval_layers_unflagged"] + phase["retrieval_layers_flagged"]) / step_ms_attr}
    attn_full_ms = mean(t_full)
    att_full_gbs = full_bytes / (attn_full_ms / 1e3) / 1e9
    roofline_attn = {"kernel": "attn_full_tc_kernel (full-cache layers: store_cache + split-K flash-decode, one launch)",
                     "bound": "hbm", "achieved": att_full_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": att_full_gbs / hbm_peak, "traffic": fa_tr["per_launch"] if fa_tr else None,
                     "bytes_per_launch": full_bytes,
                     "ms_per_launch": attn_full_ms, "peak_source": peak_src,
                     "share_of_step": phase["full_cache_layers"] / step_ms_attr}
    flag_extra_ms = sum(t_flg) - len(t_flg) * mean(t_unf)
    gather_gbs = h2d_bytes / (flag_extra_ms / 1e3) / 1e9 if flag_extra_ms > 0 else 0.0
    roofline_gather = {"kernel": "layer_kernel flagged-launch excess (score/select + host gather)", "bound": "host_link",
                       "achieved": gather_gbs, "peak": host_link_gbs, "unit": "GB/s",
                       "frac": gather_gbs / host_link_gbs if host_link_gbs else None,
                       "traffic": h2d_bytes / max(A, 1),
                       "share_of_step": phase["retrieval_layers_flagged"] / step_ms_attr,
                       "peak_source": "pinned 256 MiB cudaMemcpy H2D measured in this run"}
    # The retrieval-layer kernel's binding roofline is the host link, not HBM: per launch it moves
    # ret_bytes through HBM (~1 us at peak) but h2d_bytes / launches over PCIe (several us at peak).
    n_launch = max(len(t_unf) + len(t_flg), 1)
    link_bytes = h2d_bytes / n_launch
    link_gbs = link_bytes / (ret_ms / 1e3) / 1e9
    roofline = {"kernel": roofline_layer["kernel"], "bound": "host_link", "achieved": link_gbs,
                "peak": host_link_gbs, "unit": "GB/s", "frac": link_gbs / host_link_gbs if host_link_gbs else None,
                "traffic": None, "bytes_per_launch": link_bytes, "ms_per_launch": ret_ms,
                "traffic_note": "host-link bytes are counted by the kernel itself (stats bytes_h2d); the kernel's "
                                "DRAM traffic per launch (ncu --set full, profiles/r01_traffic.json, weighted by this "
                                "run's flagged/unflagged mix) is roofline_layer_hbm.traffic",
                "lower_bound_us": {"hbm": ret_bytes / (hbm_peak * 1e9) * 1e6,
                                   "host_link": link_bytes / (host_link_gbs * 1e9) * 1e6 if host_link_gbs else None},
                "peak_source": "pinned 256 MiB cudaMemcpy H2D measured in this run",
                "share_of_step": roofline_layer["share_of_step"]}
    retr_ms_total = flag_extra_ms

    retrievals = st_b["retrievals"] - st_a["retrievals"]
    n_ret_layers = L - len(full)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if heads else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded, planted clusters/segments; no weights on this path)",
        "config": {"workload": f"{cfg.name}: Llama-3.1-8B attention shape (L=32, Hq=32, Hkv=8, d=128), "
                               f"{cfg.prompt_len}-token prompt, S={cfg.sink_tokens} W={cfg.window_tokens} "
                               f"B={cfg.budget_tokens} tau={cfg.tau} c={cfg.avg_cluster_size}, layers 0-1 full cache",
                   "global_batch": b * jobs, "seq_len": cfg.prompt_len,
                   "parallelism": (f"kv-head shard x{world} (heads [{hb}, {hb + hc}) on rank {rank}; NCCL "
                                   f"all-gather of the per-head outputs after every layer)") if heads else
                                  f"weak dp{world} (independent sequences per rank, no collective)",
                   "l2": (f"inputs larger than L2: {kv_step_bytes / 1e6:.0f} MB of KV read per step per rank > 2 x 126 MB"
                          if flush_buf is None else
                          f"L2 flushed between steps ({kv_step_bytes / 1e6:.0f} MB of KV per step per rank; "
                          f"per-step event pairs, flush outside the timed spans)"),
                   "cuda_graph": True},
        "e2e": e2e,
        "gpu_launches": launches_per_step * K,
        "clocks": clk,
        "roofline": roofline,
        "roofline_layer_hbm": roofline_layer,
        "roofline_full_cache": roofline_attn,
        "roofline_gather": roofline_gather,
        "phases_ms_per_step": phase,
        "layer_us": layer_us,
        "kmeans_keys_per_s": km_keys / (km_ms / 1e3) if km_ms > 0 else None,
        "kmeans": {"ms_total": km_ms, "keys": km_keys, "iters": cfg.kmeans_iters,
                   "impl": "tcgen05" if args.kmeans_impl == 0 else "simt",
                   "timed": "all layers' cluster_prompt (k-means + cluster-major offload to the pinned pool; full-cache "
                            "layers: device copy) up to louiskv_prompt_fence, one event pair",
                   "prompt_offload_bytes": st0["bytes_d2h"],
                   "prompt_offload_gbs": st0["bytes_d2h"] / (km_ms / 1e3) / 1e9 if km_ms > 0 else None},
        "retrieve_us_per_step": {"per_flagged_layer_call": (retr_ms_total * 1e3 / max(1, st_d['retrievals'] - st_c['retrievals'])),
                                 "amortized_per_step": flag_extra_ms * 1e3 / max(A, 1)},
        "retrievals_per_step": retrievals / K / max(n_ret_layers, 1) / b,
        "stats_timed": {k_: st_b[k_] - st_a[k_] for k_ in st_b},
        "host_link_h2d_gbs": host_link_gbs,
        "memory": dict(ctx.memory(), full_kv_bytes=b * hc * L * (cfg.prompt_len + T) * 512,
                       note="device_bytes: every device allocation of the context (sinks, working sets, local "
                            "buffers, centroids, unit tables, the two full-cache layers, scratch); full_kv_bytes: "
                            "the K+V bf16 of every layer at P + max decode steps (a full-cache engine's device "
                            "footprint); the offloaded rows live in the pinned host pool (P:404-425)"),
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        s = oracle_sample(cfg, args.seed, args.cpu_steps)
        line["cpu_baseline"] = {"value": b / s["step_s"], "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": (f"{args.cpu_steps} decode steps of 1 retrieval-layer instance (1 KV head, "
                                           f"{g} q heads) + 1 full-cache instance at {cfg.name} sizes, extrapolated "
                                           f"x{s['n_ret']} / x{s['n_full']} instances to one 32-layer step")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
