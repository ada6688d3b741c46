#!/usr/bin/env python
"""LouisKV retrieval hot path on B200 — benchmark (driver contract: one JSON line).

Workloads (BASELINE.json configs; default C2 = configs[1], the one the metric is
quoted on): C2 Llama-3.1-8B attention shape, 32K prompt, batch 1 (long-input); C3 Qwen3-8B shape, 1K
prompt + 32K generation (short-input long-output); C4 Qwen3-8B shape, 64K prompt + 16K generation,
batch 8 (long-input long-output). Synthetic seeded data (synth/): throughput seeds plant k/4 key
groups scattered over positions (overlapping clusters). There are no weights on this path.

One timed "step" = one decode step through all L layers in model order, each layer ONE
louiskv_decode_layer call (retrieval layer: trigger -> [score / select / gather] -> store_cache ->
attention in one clustered launch; full-cache layer: store_cache + dense attention in one launch),
replayed as one CUDA graph per step with inputs already resident in HBM. The decode state is
checkpointed (louiskv_state_save) before the timed steps, so the end-to-end run (host inputs copied
in and outputs copied out every step), the L2-pressure variant and the per-kernel attribution pass
all replay EXACTLY the timed steps (same retrievals). The prompt clustering (cluster_prompt, once
per layer) is timed with the library's phase timer: k-means keys/s (Lloyd only) and the assignment
GEMM's TFLOP/s, with the prompt offload reported separately.

Multi-GPU (torchrun): --shard batch (weak scaling: every rank its own sequences, no collective) or
--shard heads (the default at N > 1 for C4 and C5: ranks own contiguous KV-head ranges of the same batch;
one NCCL all-gather of the per-head outputs per layer, or one per step with --gather step).
``--impl reference`` times the CPU oracle (the reference arm of this tier) on the box's host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "decode tok/s with LouisKV retrieval at 32K ctx; k-means keys/s; retrieve µs/step"
UNIT = "tok/s"
L2_BYTES = 126 * 2 ** 20
MODEL = {"C1": "single KV head (BASELINE configs[0])", "C2": "Llama-3.1-8B attention shape",
         "C3": "Qwen3-8B attention shape", "C4": "Qwen3-8B attention shape", "C5": "Qwen3-32B attention shape"}
PATTERN = {"C2": "long-input short-output", "C3": "short-input long-output", "C4": "long-input long-output",
           "C5": "long-input", "C1": "oracle-size case"}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=256)
    p.add_argument("--warmup", type=int, default=16)
    p.add_argument("--impl", default="product", choices=["product", "reference"])
    p.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5"])
    p.add_argument("--shard-of", type=int, default=0,
                   help="N > 1 at one GPU: run rank 0's share of an N-GPU KV-head-sharded job (its KV heads "
                        "[0, Hkv/N) of every sequence; the all-gather is not run) — C5's per-GPU work")
    p.add_argument("--batch", type=int, default=0, help="override the config's batch (host-memory bound)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-l2-variant", action="store_true")
    p.add_argument("--kmeans-impl", type=int, default=0)
    p.add_argument("--max-output-len", type=int, default=0,
                   help="context capacity for generated tokens (default: the config's own generation length)")
    p.add_argument("--shard", default="auto", choices=["auto", "batch", "heads"],
                   help="multi-GPU partitioning: 'batch' = every rank its own sequences (weak scaling, no "
                        "collective); 'heads' = ranks own contiguous KV-head ranges of the same sequences and "
                        "all-gather the per-head attention outputs over NCCL (strong scaling); auto = heads for "
                        "C4 and C5 at N > 1, else batch")
    p.add_argument("--gather", default="layer", choices=["layer", "step"],
                   help="heads mode: one all-gather per layer (model-faithful) or one batched per step")
    return p.parse_args(argv)


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
                 "-lms", "50"], stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
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
    """All-gather of per-head attention outputs (north_star: NCCL over NVLink, only for the outputs).
    out_own [..., b, g*hc, d] -> gathered [world, ..., b, g*hc, d] (rank-major). Stream-ordered, so it
    is captured into the step's CUDA graph. Works for one layer ([b, gq, d]) or a whole step
    ([L, b, gq, d], the per-step batched variant)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_gather_into_tensor(gathered.view((-1,) + tuple(out_own.shape[1:])), out_own)
    else:
        gathered[0].copy_(out_own)


def assemble_heads(gathered):
    """[world, b, g*hc, d] -> [b, Hq, d] in model head order (what the O-projection consumes); a step's
    [world, L, b, g*hc, d] -> [L, b, Hq, d]."""
    if gathered.dim() == 5:
        w, L, b, gh, d = gathered.shape
        return gathered.permute(1, 2, 0, 3, 4).reshape(L, b, w * gh, d)
    w, b, gh, d = gathered.shape
    return gathered.permute(1, 0, 2, 3).reshape(b, w * gh, d)


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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def n_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


CONFIG_BATCH = {"C1": 1, "C2": 1, "C3": 1, "C4": 8, "C5": 32}


def throughput_cfg(name: str):
    """The config as benchmarked: throughput seeds plant k/4 key groups."""
    from synth.configs import CONFIGS
    cfg = CONFIGS[name]
    return cfg.replace(k_planted=max(cfg.n_clusters // 4, 2 * cfg.n_targets))


def workload_label(cfg, T_steps=None) -> str:
    full = ",".join(str(l) for l in cfg.full_cache_layers)
    return (f"{cfg.name} {PATTERN.get(cfg.name, '')}: {MODEL.get(cfg.name, cfg.name)} (L={cfg.num_layers}, "
            f"Hq={cfg.num_q_heads}, Hkv={cfg.num_kv_heads}, d={cfg.head_dim}), {cfg.prompt_len}-token prompt, "
            f"{cfg.decode_steps}-token generation, batch {cfg.batch}, S={cfg.sink_tokens} W={cfg.window_tokens} "
            f"B={cfg.budget_tokens} tau={cfg.tau} c={cfg.avg_cluster_size}, full-cache layers {full}; "
            f"k-means {cfg.kmeans_iters} iters; planted key groups k/4 = {cfg.k_planted}")


def table3_accounting(cfg, hc, m_out):
    """GPU KV footprint, Table 3: FullCache 4 L h d (n + m), LouisKV 4 L h d (B + n/(2c) +
    m/(2s)) bytes (fp16 K+V, one fp16 index vector per cluster / segment), for this rank's heads and
    the whole batch, with s = the config's mean segment length; next to it the same quantities as this
    build keeps them (retrieval layers: sinks S + double-buffered working set 2B + local buffer W rows
    of K+V bf16, one fp32 master + one bf16 copy per unit index at the unit-table capacity; full-cache
    layers: everything)."""
    L, Lf = cfg.num_layers, len(cfg.full_cache_layers)
    n, m, B, c, s_ = cfg.prompt_len, m_out, cfg.budget_tokens, cfg.avg_cluster_size, cfg.seg_mean
    hd = hc * cfg.head_dim * cfg.batch
    full = 4 * L * hd * (n + m)
    louis = 4 * L * hd * (B + n / (2 * c) + m / (2 * s_))
    units_cap = -(-((n - cfg.sink_tokens) // c + m) // 256) * 256
    ours = (4 * (L - Lf) * hd * (cfg.sink_tokens + 2 * B + cfg.window_tokens + 2)
            + (L - Lf) * hd * units_cap * (4 + 2)
            + 4 * Lf * hd * (n + m))
    return {"fullcache_formula_bytes": full, "louiskv_formula_bytes": louis, "build_kv_state_bytes": ours,
            "build_over_formula": ours / louis,
            "note": "the build's excess over the formula: the first two layers kept in full (P:143; not in "
                    "Table 3), the double-buffered working set, sinks and local buffer, and fp32 + bf16 unit "
                    "indices sized to capacity (the formula counts one fp16 vector per unit)"}


# ----------------------------------------------------------------------------- oracle (CPU) legs
# Only bench's cpu_baseline leg and --impl reference execute anything under oracle/ (tier rule ③).
def _oracle_worker(args):
    """One process: run the oracle decode (Algorithm 1 order per instance) for the given
    (layer, kv-head) instances over `steps` steps. Returns seconds per phase of the run."""
    (cfg_name, kp, seed, insts, steps, warm, start_evt, plen) = args
    import numpy as np
    import torch
    import synth
    from synth.configs import CONFIGS
    from oracle.episode import OracleEpisode
    from _pair import planted_assign
    torch.set_num_threads(1)
    cfg = CONFIGS[cfg_name].replace(k_planted=kp)
    if plen:
        cfg = cfg.replace(prompt_len=plen, k_planted=kp)
    T = warm + steps
    layers = sorted({l for l, _ in insts})
    plants = {l: synth.planted(cfg, l, seed, "cpu") for l in layers}
    eps = {}
    for l, h in insts:
        ep = OracleEpisode(cfg, kv_head_begin=h, kv_head_count=1)
        K, V, lab = synth.prompt_kv(cfg, l, seed, "cpu", plants[l], return_labels=True)
        Kn = K[:, :, h:h + 1].float().numpy()
        Vn = V[:, :, h:h + 1].float().numpy()
        if l in cfg.full_cache_layers:
            ep.cluster_prompt(l, Kn, Vn)
        else:
            ep.cluster_prompt(l, Kn, Vn, assign=planted_assign(cfg, lab[:, :, h:h + 1]))
        eps[(l, h)] = ep
    # decode inputs of the needed layers only (same generator as the product arm)
    one = cfg.replace(num_layers=max(layers) + 1, k_planted=kp)
    q, k, v, _ = synth.decode_stream(one, T, seed, "cpu", [plants.get(l) or synth.planted(one, l, seed, "cpu")
                                                           for l in range(max(layers) + 1)])
    qn, kn, vn = q.float().numpy(), k.float().numpy(), v.float().numpy()
    g = cfg.group
    if start_evt is not None:
        start_evt.wait()

    def run(t):
        for (l, h), ep in eps.items():
            ep.should_retrieve(l, qn[t, l])
            ep.retrieve(l, qn[t, l][:, h * g:(h + 1) * g])
            ep.append_output(l, kn[t, l][:, h:h + 1], vn[t, l][:, h:h + 1])
            ep.sparse_attn(l, qn[t, l][:, h * g:(h + 1) * g])

    for t in range(warm):
        run(t)
    t0 = time.perf_counter()
    for t in range(warm, T):
        run(t)
    return time.perf_counter() - t0


def _kmeans_worker(args):
    """One Lloyd iteration of the oracle k-means on one instance of the config (seconds)."""
    cfg_name, kp, seed, layer, head = args
    import synth
    import oracle
    from synth.configs import CONFIGS
    cfg = CONFIGS[cfg_name].replace(k_planted=kp)
    K, _ = synth.prompt_kv(cfg, layer, seed, "cpu")
    X = K[0, cfg.sink_tokens:, head].float().numpy().copy()
    k = cfg.n_clusters
    t0 = time.perf_counter()
    oracle.kmeans(X, k, 1, mode=1)
    return time.perf_counter() - t0


def _pool(n):
    import multiprocessing as mp
    return mp.get_context("fork").Pool(n)


def cpu_baseline(cfg, seed: int, steps: int = 12, warm: int = 2):
    """The oracle as it stands on the host cores, bounded samples of the same workload:
    decode — one retrieval-layer instance + one full-cache instance per process for `steps` steps,
    alone (1 thread) and one process per core concurrently (different instances); k-means — one Lloyd
    iteration of one instance, alone and one per core. Extrapolated to whole steps / all iterations."""
    import oracle  # noqa: F401  (builds the C oracle once before forking)
    oracle.build_oracle()
    nc = n_cores()
    full = sorted(cfg.full_cache_layers)
    ret = [l for l in range(cfg.num_layers) if l not in cfg.full_cache_layers]
    plen = 0
    t1 = _oracle_worker((cfg.name, cfg.k_planted, seed, [(ret[0], 0), (full[0], 0)], steps, warm, None, plen))
    jobs = [(cfg.name, cfg.k_planted, seed, [(ret[i % len(ret)], i % cfg.num_kv_heads),
                                             (full[i % len(full)], (i + 1) % cfg.num_kv_heads)], steps, warm, None, plen)
            for i in range(nc)]
    w0 = time.perf_counter()
    with _pool(nc) as p:
        tn = p.map(_oracle_worker, jobs)
    wall = time.perf_counter() - w0
    # per-step work of the full config: n_ret retrieval + n_full full-cache instance-steps; the pair
    # sample is split into its parts with a second 1-thread sample of the retrieval instance alone
    n_ret = cfg.batch * len(ret) * cfg.num_kv_heads
    n_full = cfg.batch * len(full) * cfg.num_kv_heads
    per_pair_1t = t1 / steps  # one retrieval + one full-cache instance-step, one thread
    t_ret = _oracle_worker((cfg.name, cfg.k_planted, seed, [(ret[0], 0)], steps, warm, None, plen)) / steps
    t_full = max(per_pair_1t - t_ret, 0.0)
    step_1t = n_ret * t_ret + n_full * t_full
    # all cores: every process does 1/nc of the instances, each slowed by the measured contention
    # (mean time of the concurrent samples over the same sample alone)
    par_eff = (sum(tn) / len(tn)) / t1
    step_nc = step_1t * par_eff / nc
    # k-means: one iteration of one instance
    kt1 = _kmeans_worker((cfg.name, cfg.k_planted, seed, ret[0], 0))
    w0 = time.perf_counter()
    with _pool(nc) as p:
        ktn = p.map(_kmeans_worker, [(cfg.name, cfg.k_planted, seed, ret[i % len(ret)], i % cfg.num_kv_heads)
                                     for i in range(nc)])
    kwall = time.perf_counter() - w0
    N = cfg.prompt_len - cfg.sink_tokens
    return {
        "value": cfg.batch / (step_nc if nc > 1 else step_1t), "unit": UNIT, "cores": nc, "kind": "oracle",
        "cpu_model": cpu_model(),
        "value_1_thread": cfg.batch / step_1t,
        "ms_per_step_1_thread": step_1t * 1e3, "ms_per_step_all_cores": step_nc * 1e3,
        "per_instance_step_ms": {"retrieval": t_ret * 1e3, "full_cache": t_full * 1e3},
        "concurrent_slowdown": par_eff, "concurrent_wall_s": wall,
        "kmeans_keys_per_s_1_thread": N / (kt1 * cfg.kmeans_iters),
        "kmeans_keys_per_s_all_cores": nc * N / (max(ktn) * cfg.kmeans_iters),
        "kmeans_iter_s_1_thread": kt1, "kmeans_wall_s_all_cores": kwall,
        "sample": (f"decode: {steps} steps ({warm} warm-up) of one retrieval-layer + one full-cache instance "
                   f"(1 KV head, {cfg.group} q heads) at {cfg.name} sizes, alone (1 thread) and one process per "
                   f"core concurrently ({nc} processes, different instances), extrapolated x{n_ret} retrieval / "
                   f"x{n_full} full-cache instances to one {cfg.num_layers}-layer step (all cores: x parallel "
                   f"efficiency / {nc}); k-means: one Lloyd iteration (N={N}, k={cfg.n_clusters}, d=128, fp64) of "
                   f"one instance alone and {nc} concurrently, x{cfg.kmeans_iters} iterations"),
    }


def run_reference(args):
    """--impl reference: the CPU oracle, as it stands, on the box's host cores (rank 0 only). C2: FULL
    decode steps — every (layer, kv-head) instance of the config, spread over one process per core;
    C3/C4: a sample of instances (stated), extrapolated by instance count."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    import oracle
    oracle.build_oracle()
    cfg = throughput_cfg(args.config)
    nc = n_cores()
    L, H = cfg.num_layers, cfg.num_kv_heads
    all_inst = [(l, h) for l in range(L) for h in range(H)]
    if cfg.name == "C2":
        chosen, scale, kind = all_inst, 1.0, "full steps"
    else:
        # sample: every layer kind, one KV head per layer, batch as configured
        chosen = [(l, l % H) for l in range(L)]
        scale, kind = len(all_inst) / len(chosen), f"sampled {len(chosen)} of {len(all_inst)} (layer, kv-head) instances"
    # balance: full-cache instances (expensive) dealt first, round robin
    full = [i for i in chosen if i[0] in cfg.full_cache_layers]
    rest = [i for i in chosen if i[0] not in cfg.full_cache_layers]
    nw = min(nc, len(chosen))
    buckets = [[] for _ in range(nw)]
    for j, inst in enumerate(full + rest):
        buckets[j % nw].append(inst)
    K, W = max(args.steps, 1), max(args.warmup, 0)
    t0 = time.perf_counter()
    with _pool(nw) as p:
        times = p.map(_oracle_worker, [(cfg.name, cfg.k_planted, args.seed, bk, K, W, None, 0) for bk in buckets])
    wall = time.perf_counter() - t0
    step_s = max(times) / K * scale  # the slowest process bounds a step
    value = cfg.batch / step_s
    sample = (f"{kind}: {len(chosen)} instances of {cfg.name} (batch {cfg.batch}) on {nw} processes "
              f"(one per core), {W} warm-up + {K} timed decode steps each; step time = slowest process"
              + ("" if scale == 1.0 else f", x{scale:.1f} instances (extrapolated)"))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "warmup": W, "ms_per_step": step_s * 1e3, "ms_per_step_extrapolated": scale != 1.0,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, planted clusters/segments; the product arm's recipe, CPU random stream)",
            "config": {"workload": workload_label(cfg), "global_batch": cfg.batch, "seq_len": cfg.prompt_len},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": nw, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- product leg
def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import synth
    import paper_2510_11292_b200 as lkv

    world, rank, local = dist_setup()
    dev = torch.device("cuda", local)
    cfg = throughput_cfg(args.config)
    if args.batch:
        cfg = cfg.replace(batch=args.batch, k_planted=cfg.k_planted)
    L, b, Hq, Hkv, d, g = cfg.num_layers, cfg.batch, cfg.num_q_heads, cfg.num_kv_heads, cfg.head_dim, cfg.group
    full = set(cfg.full_cache_layers)
    ret_layers = [l for l in range(L) if l not in full]
    K, W = args.steps, args.warmup
    T = 1 + W + K + 2
    shard = args.shard if args.shard != "auto" else ("heads" if (world > 1 and cfg.name in ("C4", "C5")) else "batch")
    heads = shard == "heads"
    seed = args.seed if heads else rank_seed(args.seed, rank)
    hb, hc = head_range(rank, world, Hkv) if heads else (0, Hkv)
    if args.shard_of > 1 and world == 1:
        hb, hc = head_range(0, args.shard_of, Hkv)
    gq = g * hc
    jobs = 1 if heads else world
    cap_out = args.max_output_len or max(cfg.max_output_len, T + 1)
    ctx = lkv.Context(lkv.make_config(cfg, kv_head_begin=hb, kv_head_count=hc, max_output_len=cap_out, device=local,
                                      kmeans_impl=args.kmeans_impl))
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"

    # ---------------- prefill: cluster_prompt per layer (inputs generated per layer, so C4's 73 GB
    # prompt never sits on the device at once); phase timer on
    ctx.set_prefill_timing(True)
    plants = [synth.planted(cfg, l, seed, dev) for l in range(L)]
    km_ms_calls = 0.0
    km_keys = 0
    for l in range(L):
        Kl, Vl = synth.prompt_kv(cfg, l, seed, dev, plants[l])
        Kl, Vl = Kl[:, :, hb:hb + hc], Vl[:, :, hb:hb + hc]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.cluster_prompt(l, Kl, Vl)
        e1.record()
        torch.cuda.synchronize()
        km_ms_calls += e0.elapsed_time(e1)
        if l not in full:
            km_keys += b * hc * (cfg.prompt_len - cfg.sink_tokens)
        del Kl, Vl
    ctx.prompt_fence()
    torch.cuda.synchronize()
    pt = ctx.prefill_times()
    ctx.set_prefill_timing(False)
    st0 = ctx.stats()

    # ---------------- decode inputs (device resident) and static graph buffers
    q, kk, vv, _ = synth.decode_stream(cfg, T, seed, dev, plants)
    del plants
    n_q, n_kv = L * b * Hq * d, L * b * Hkv * d
    qkv = torch.cat([q.reshape(T, -1), kk.reshape(T, -1), vv.reshape(T, -1)], dim=1)
    del q, kk, vv
    qkv_in = torch.empty((n_q + 2 * n_kv,), dtype=torch.bfloat16, device=dev)
    out = torch.empty((L, b, gq, d), dtype=torch.bfloat16, device=dev)
    gathered = torch.empty((world, L, b, gq, d), dtype=torch.bfloat16, device=dev) if heads else None
    flags = torch.zeros((L, b), dtype=torch.uint8, device=dev)

    def views(src):
        qs = src[:n_q].view(L, b, Hq, d)
        ks = src[n_q:n_q + n_kv].view(L, b, Hkv, d)[:, :, hb:hb + hc]
        vs = src[n_q + n_kv:].view(L, b, Hkv, d)[:, :, hb:hb + hc]
        return qs, ks, vs

    def issue_layers(layers, src=None, between=None):
        qs, ks, vs = views(qkv_in if src is None else src)
        for l in layers:
            ctx.decode_layer(l, qs[l], ks[l], vs[l], out[l], flag_out=flags[l])
            if heads and args.gather == "layer":
                gather_heads(out[l], gathered[:, l], world)
            if between is not None:
                between()
        if heads and args.gather == "step" and len(layers) == L:
            gather_heads(out, gathered, world)

    def issue_step(src=None, between=None):
        issue_layers(range(L), src, between)

    step_idx = 0
    qkv_in.copy_(qkv[step_idx])
    issue_step()  # step 1 runs directly (t == 1: retrieval everywhere)
    step_idx += 1
    torch.cuda.synchronize()
    cap_stream = torch.cuda.Stream(device=dev)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=cap_stream):
        issue_step()
    for _ in range(W):
        qkv_in.copy_(qkv[step_idx])
        graph.replay()
        step_idx += 1
    s0 = step_idx  # first timed step
    step_graphs = []
    for i in range(K):
        gi = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gi, stream=cap_stream):
            issue_step(src=qkv[s0 + i])
        step_graphs.append(gi)
    torch.cuda.synchronize()
    ctx.state_save()  # the timed steps are replayed exactly by e2e / L2 / attribution below
    torch.cuda.synchronize()

    # ---------------- timed region (device-resident inputs)
    P_ = cfg.prompt_len
    kv_step_bytes = (len(full) * b * hc * (P_ + s0) + len(ret_layers) * b * hc *
                     (cfg.sink_tokens + cfg.budget_tokens + cfg.window_tokens)) * 512
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if kv_step_bytes < 2 * L2_BYTES else None

    def dev_timed(body, n):
        """Device time of n calls of body(i); L2 flushed between steps (outside the timed spans) when the
        rank's per-step KV bytes fit in L2."""
        if flush_buf is None:
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            for i in range(n):
                body(i)
            t1.record()
            torch.cuda.synchronize()
            return t0.elapsed_time(t1)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            flush_buf.add_(1)
            evs[i][0].record()
            body(i)
            evs[i][1].record()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(z) for a, z in evs)

    clocks = ClockSampler(local)
    barrier(world)
    clocks.start()
    st_a = ctx.stats()
    barrier(world)
    ms = dev_timed(lambda i: step_graphs[i].replay(), K)
    barrier(world)
    clk = clocks.stop()
    ms = max_over_ranks(ms, world)
    st_b = ctx.stats()
    stats_timed = {k_: st_b[k_] - st_a[k_] for k_ in st_b if not k_.startswith("kmeans")}
    value = jobs * b * K / (ms / 1e3)
    del step_graphs

    # ---------------- e2e: the SAME steps again from the checkpoint, host inputs -> device, graph,
    # outputs -> host, every step (through the public API: louiskv_decode_layer per layer)
    ctx.state_restore()
    qkv_h = qkv[s0:s0 + K].cpu().pin_memory()
    res = gathered if heads else out
    oh = torch.empty((K,) + tuple(res.shape), dtype=torch.bfloat16).pin_memory()
    barrier(world)

    def e2e_body(i):
        qkv_in.copy_(qkv_h[i], non_blocking=True)
        graph.replay()
        oh[i].copy_(res, non_blocking=True)

    st_e0 = ctx.stats()
    e2e_ms = dev_timed(e2e_body, K)
    barrier(world)
    st_e1 = ctx.stats()
    e2e_ms = max_over_ranks(e2e_ms, world)
    e2e = {"value": jobs * b * K / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": int(qkv_h[0].numel()) * 2, "d2h_bytes_per_step": int(oh[0].numel()) * 2,
           "ms_per_step": e2e_ms / K, "same_steps_as_value": True,
           "retrievals_same": (st_e1["retrievals"] - st_e0["retrievals"]) == stats_timed["retrievals"]}
    del qkv_h, oh

    # ---------------- L2-pressure variant: the same steps with a 2 x L2 buffer rewritten between layers
    # (stand-in for the weight traffic of a real model between attention layers; no PDL edge across it);
    # attention-side time = (steps with flushes) - (the flushes alone)
    l2v = None
    if not args.no_l2_variant:
        ctx.state_restore()
        fl_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        gl2, gfl = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(gl2, stream=cap_stream):
            issue_step(between=lambda: fl_buf.add_(1))
        with torch.cuda.graph(gfl, stream=cap_stream):
            for _ in range(L):
                fl_buf.add_(1)
        K2 = K

        def l2_body(i):
            qkv_in.copy_(qkv[s0 + i], non_blocking=True)
            gl2.replay()

        def fl_body(i):
            qkv_in.copy_(qkv[s0 + i], non_blocking=True)
            gfl.replay()

        ms_l2 = max_over_ranks(dev_timed(l2_body, K2), world)
        ms_fl = max_over_ranks(dev_timed(fl_body, K2), world)
        att_ms = (ms_l2 - ms_fl) / K2
        l2v = {"ms_per_step_with_flushes": ms_l2 / K2, "flush_ms_per_step": ms_fl / K2,
               "attention_side_ms_per_step": att_ms, "value": jobs * b / (att_ms / 1e3),
               "unit": UNIT, "flush_bytes_per_layer": 2 * fl_buf.numel() * 4,
               "note": "same timed steps (checkpoint restore); a 252 MB read+write between every two layers "
                       "evicts L2, so every layer starts cold; value = attention-side tok/s"}
        del gl2, gfl, fl_buf

    # ---------------- attribution: the same steps again, the retrieval layers and the full-cache layers
    # as two graphs (each replay timed on the device); least squares on the per-replay flag counts
    ctx.state_restore()
    g_ret, g_full = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_ret, stream=cap_stream):
        issue_layers(ret_layers)
    with torch.cuda.graph(g_full, stream=cap_stream):
        issue_layers(sorted(full))
    rows_fit, t_full = [], []
    st_c = ctx.stats()
    for i in range(K):
        qkv_in.copy_(qkv[s0 + i])
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
    full_ms = float(np.mean(t_full)) if full else 0.0
    ret_ms_attr = float(y.mean())  # retrieval layers per step (attribution replays)
    layer_us = {"retrieval_unflagged": u_ms * 1e3, "retrieval_flagged": f_ms * 1e3, "full_cache": full_ms * 1e3,
                "n_flagged_launches": n_flg_tot, "n_unflagged_launches": n_unf_tot,
                "method": "the timed steps replayed from the checkpoint as a retrieval-layers-only graph and a "
                          "full-cache-layers-only graph, each replay timed on the device; flagged / unflagged "
                          "per-launch time by least squares on the per-replay flag counts"}

    # ---------------- host-link peak (pinned H2D copy)
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

    # ---------------- rooflines, from the TIMED window: the full-cache layers' share is their
    # attribution time (flag independent), the retrieval layers get the rest of the timed step
    ms_step = ms / K
    full_ms_step = full_ms * len(full)
    ret_ms_step = max(ms_step - full_ms_step, 1e-9)
    n_ret_launch = len(ret_layers) * K
    # algorithmic bytes of the retrieval-layer launches over the timed window: attended rows (sinks +
    # working set + local buffer, from the unit tables at the window's end, 512 B each) per launch, plus
    # on flagged launches the centroid reads (units scored x 256 B) and the working-set rebuild
    # (new rows read over the link and written, kept rows read and written: <= B rows per instance)
    att_rows = 0
    kc = cfg.n_clusters
    t_end = s0 + K
    for l in ret_layers:
        for bb in range(b):
            for hh in range(hc):
                _, sizes, _ = ctx.get_units(l, bb, hh)
                nws = len(ctx.get_working_set(l, bb, hh)[0])
                att_rows += min(cfg.sink_tokens, P_) + nws + max(0, t_end - int(sizes[kc:].sum()))
    att_bytes_launch = att_rows / max(len(ret_layers), 1) * 512
    ret_bytes = att_bytes_launch * n_ret_launch + stats_timed["units_scored"] * 256 + stats_timed["bytes_h2d"]
    # working-set rows written per retrieval (upper bound: B rows per (sequence, owned head))
    ws_rebuild = stats_timed["retrievals"] * hc * cfg.budget_tokens * 512
    ret_bytes += ws_rebuild
    ret_gbs = ret_bytes / (ret_ms_step * K / 1e3) / 1e9
    link_bytes = stats_timed["bytes_h2d"]
    link_gbs = link_bytes / (ret_ms_step * K / 1e3) / 1e9
    full_bytes_launch = b * hc * (P_ + s0 + K // 2) * 2 * d * 2
    full_gbs = full_bytes_launch / (full_ms / 1e3) / 1e9 if full_ms > 0 else 0.0
    share_ret, share_full = ret_ms_step / ms_step, full_ms_step / ms_step
    roof_layer_link = {"kernel": "layer_kernel (retrieval layers: trigger + score/select + host gather + append + "
                                 "attention, one clustered launch)",
                       "bound": "host_link", "achieved": link_gbs, "peak": host_link_gbs, "unit": "GB/s",
                       "frac": link_gbs / host_link_gbs if host_link_gbs else None, "traffic": None,
                       "bytes_per_launch": link_bytes / max(n_ret_launch, 1),
                       "ms_per_launch": ret_ms_step / max(len(ret_layers), 1),
                       "peak_source": "pinned 256 MiB cudaMemcpy H2D measured in this run",
                       "share_of_step": share_ret,
                       "note": "timed window: host-pool bytes the gathers read (kernel stats) / the retrieval "
                               "layers' share of the timed step time"}
    roof_layer_hbm = {"kernel": roof_layer_link["kernel"], "bound": "hbm", "achieved": ret_gbs, "peak": hbm_peak,
                      "unit": "GB/s", "frac": ret_gbs / hbm_peak, "traffic": None,
                      "bytes_per_launch": ret_bytes / max(n_ret_launch, 1),
                      "ms_per_launch": ret_ms_step / max(len(ret_layers), 1), "peak_source": peak_src,
                      "share_of_step": share_ret}
    roof_full = {"kernel": "attn_full_tc_kernel (full-cache layers: store_cache + split-K flash-decode, one launch)",
                 "bound": "hbm", "achieved": full_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": full_gbs / hbm_peak,
                 "traffic": None, "bytes_per_launch": full_bytes_launch, "ms_per_launch": full_ms,
                 "peak_source": peak_src, "share_of_step": share_full}
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(cfg.name, {})
    except Exception:
        tr = {}
    if "attn_full_tc_kernel" in tr:
        roof_full["traffic"] = tr["attn_full_tc_kernel"]
    if "layer_kernel" in tr:
        roof_layer_hbm["traffic"] = tr["layer_kernel"]
    # the flagged launches alone against the host link (the resource a retrieval is bound by): the
    # attribution pass's host-pool bytes ÷ (flagged launches × the fitted flagged-launch time)
    h2d_attr = st_d["bytes_h2d"] - st_c["bytes_h2d"]
    fl_gbs = h2d_attr / (n_flg_tot * f_ms / 1e3) / 1e9 if n_flg_tot and f_ms > 0 else 0.0
    flagged_link = {"kernel": "layer_kernel, flagged launches (trigger + score/select + host gather + append + "
                              "attention)", "bound": "host_link", "achieved": fl_gbs, "peak": host_link_gbs,
                    "unit": "GB/s", "frac": fl_gbs / host_link_gbs if host_link_gbs else None,
                    "bytes_per_flagged_launch": h2d_attr / max(n_flg_tot, 1), "us_per_flagged_launch": f_ms * 1e3,
                    "note": "counter-backed: ncu pcie__read_bytes on flagged launches, profiles/r02_ncu_summary.md"}
    # the dominant kernel's binding resource: of the host link and HBM, the one whose lower-bound time
    # for the measured bytes is larger (C2 / C4: the link; C3, where retrievals move few host bytes:
    # HBM — the kernel is latency-bound there)
    lb_link = link_bytes / (host_link_gbs * 1e9) if host_link_gbs else 0.0
    lb_hbm = ret_bytes / (hbm_peak * 1e9)
    roof_layer = roof_layer_link if lb_link >= lb_hbm else roof_layer_hbm
    roof_layer["binding"] = {"host_link_lower_bound_ms": lb_link * 1e3, "hbm_lower_bound_ms": lb_hbm * 1e3}
    dominant = roof_full if share_full > share_ret else roof_layer
    # k-means: the assignment GEMM (tensor pipe) and the Lloyd loop, from the phase timer
    lloyd_ms = pt["init_ms"] + pt["assign_ms"] + pt["sort_ms"] + pt["update_ms"]
    gemm_tf = pt["assign_flops"] / (pt["assign_ms"] / 1e3) / 1e12 if pt["assign_ms"] > 0 else 0.0
    tf_sus = peaks.get("bf16_tflops_sustained", 1364.5)
    tf_burst = peaks.get("bf16_tflops", 1604.9)
    roof_km = {"kernel": "kmeans_assign_tc_kernel (tcgen05 GEMM X.C^T + fused argmax epilogue)", "bound": "tensor",
               "achieved": gemm_tf, "peak": tf_sus, "unit": "TFLOP/s", "frac": gemm_tf / tf_sus,
               "frac_of_burst_peak": gemm_tf / tf_burst, "traffic": None,
               "flops": pt["assign_flops"], "ms": pt["assign_ms"], "passes": pt["assign_passes"],
               "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (the prefill runs for tens of ms to "
                              "seconds); frac_of_burst_peak against bf16_tflops",
               "note": "algorithmic flops 2 N k d per instance-iteration / device time of the assignment passes "
                       "(CUDA events of the library's prefill phase timer)"}
    kmeans = {"keys_per_s_lloyd": pt["keys"] / (lloyd_ms / 1e3) if lloyd_ms > 0 else None,
              "keys_per_s_incl_offload_staging": km_keys * jobs / (km_ms_calls / 1e3) if km_ms_calls > 0 else None,
              "iters": cfg.kmeans_iters, "keys": pt["keys"],
              "phase_ms": {k_: pt[k_] for k_ in ("init_ms", "assign_ms", "sort_ms", "update_ms", "stage_ms", "d2h_ms")},
              "non_gemm_share_of_iteration": (pt["sort_ms"] + pt["update_ms"]) / max(pt["assign_ms"] + pt["sort_ms"] +
                                                                                    pt["update_ms"], 1e-9),
              "offload": {"bytes": pt["d2h_bytes"], "d2h_ms": pt["d2h_ms"],
                          "gbs": pt["d2h_bytes"] / (pt["d2h_ms"] / 1e3) / 1e9 if pt["d2h_ms"] > 0 else None,
                          "note": "copy-engine D2H of the cluster-major rows into the pinned pool, on the "
                                  "library's copy stream (overlaps the next layer's clustering)"},
              "impl": "tcgen05" if args.kmeans_impl == 0 else "simt"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong" if heads else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded; k/4 planted key groups scattered over positions, planted query segments; "
                "no weights on this path)",
        "config": {"workload": workload_label(cfg), "global_batch": b * jobs, "seq_len": cfg.prompt_len,
                   "decode_window": f"steps t = {s0 + 1}..{s0 + K} of the generation (after {W} warm-up steps)",
                   "capacity_max_output_len": cap_out,
                   **({"batch_override": f"batch {b} instead of the config's {CONFIG_BATCH[cfg.name]}: the pinned pool "
                                         f"of the full batch exceeds this box's host memory"}
                      if args.batch else {}),
                   "parallelism": ((f"one rank's share of a {args.shard_of}-GPU KV-head shard: heads [{hb}, {hb + hc}) "
                                    f"of {Hkv} (the all-gather of the per-head outputs is not run at one GPU)")
                                   if args.shard_of > 1 and world == 1 else
                                   (f"kv-head shard x{world} (heads [{hb}, {hb + hc}) on rank {rank}; NCCL all-gather "
                                    f"of the per-head outputs {'per layer' if args.gather == 'layer' else 'once per step'})")
                                   if heads else f"weak dp{world} (independent sequences per rank, no collective)"),
                   "l2": (f"inputs larger than L2: {kv_step_bytes / 1e6:.0f} MB of KV read per step per rank > 2 x 126 MB"
                          if flush_buf is None else
                          f"L2 flushed between steps ({kv_step_bytes / 1e6:.0f} MB of KV per step per rank)"),
                   "cuda_graph": True},
        "e2e": e2e,
        "gpu_launches": L * K,
        "clocks": clk,
        "roofline": dominant,
        "roofline_layer_link": roof_layer_link,
        "roofline_layer_hbm": roof_layer_hbm,
        "roofline_flagged_link": flagged_link,
        "roofline_full_cache": roof_full,
        "roofline_kmeans": roof_km,
        "kmeans_keys_per_s": kmeans["keys_per_s_lloyd"],
        "kmeans": kmeans,
        "layer_us": layer_us,
        "phases_ms_per_step": {"retrieval_layers": ret_ms_step, "full_cache_layers": full_ms_step,
                               "retrieval_layers_attribution": ret_ms_attr},
        "retrieve_us_per_step": {"per_flagged_launch_excess": (f_ms - u_ms) * 1e3,
                                 "amortized_per_step": (f_ms - u_ms) * 1e3 * n_flg_tot / K},
        "retrievals_per_layer_step": stats_timed["retrievals"] / K / max(len(ret_layers), 1) / b,
        "stats_timed": stats_timed,
        "l2_pressure": l2v,
        "host_link_h2d_gbs": host_link_gbs,
        "memory": dict(ctx.memory(), full_kv_bytes=b * hc * L * (cfg.prompt_len + cap_out) * 512,
                       table3=table3_accounting(cfg, hc, cap_out),
                       note="device_bytes: every device allocation of the context; full_kv_bytes: the K+V bf16 of "
                            "every layer at P + capacity (a full-cache engine's device footprint); the offloaded "
                            "rows live in the pinned host pool (P:404-425)"),
    }
    ctx.close()
    del graph
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.seed)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
