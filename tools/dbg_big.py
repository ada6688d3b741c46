"""Debug: big-mode select of the layer kernel (n > 8192 live units) vs the oracle, one step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import test_gpu_parity as tp
from _pair import make_inputs, np32, bf16_bits
from oracle.episode import OracleEpisode
import paper_2510_11292_b200 as lkv

for prompt_len in (8000 + 16, 12000 + 16):
    cfg = tp.small_cfg(num_layers=1, full_cache_layers=(), decode_steps=8, batch=1, num_kv_heads=1, num_q_heads=4,
                       prompt_len=prompt_len, avg_cluster_size=1, budget_tokens=300, tau=0.95)
    inp = make_inputs(cfg, 8, 10)
    N = prompt_len - cfg.sink_tokens
    a = np.arange(N, dtype=np.int32)[None, None, :]
    ctx = lkv.Context(lkv.make_config(cfg))
    ep = OracleEpisode(cfg)
    Kn, Vn = np32(inp.K[0]), np32(inp.V[0])
    ep.cluster_prompt(0, Kn, Vn, assign=a)
    cen = np.stack([[np.stack([u.centroid for u in ep.units(0, 0, 0)])]])
    ctx.set_prompt_units(0, inp.K[0], inp.V[0], a, cen)
    out = torch.zeros((1, 4, 128), dtype=torch.bfloat16, device="cuda")
    out32 = torch.zeros((1, 4, 128), dtype=torch.float32, device="cuda")
    fl = torch.zeros(1, dtype=torch.uint8, device="cuda")
    for t in range(2):
        ctx.decode_layer(0, inp.q[t, 0], inp.k[t, 0].contiguous(), inp.v[t, 0].contiguous(), out, out32, fl)
        f, r = ep.should_retrieve(0, np32(inp.q[t, 0]))
        ep.retrieve(0, np32(inp.q[t, 0]))
        ep.append_output(0, np32(inp.k[t, 0]), np32(inp.v[t, 0]))
        o = ep.sparse_attn(0, np32(inp.q[t, 0]))
        torch.cuda.synchronize()
        sg = ctx.get_selection(0, 0, 0)
        so = np.array(ep.selection(0, 0, 0))
        Kw, Vw = ctx.get_working_set(0, 0, 0)
        print(prompt_len, t, "flag", int(fl.item()), f, "nsel gpu", len(sg), "oracle", len(so),
              "same", np.array_equal(sg, so), "common", len(np.intersect1d(sg, so)),
              "ws rows", len(Kw), "err", np.abs(out32.cpu().numpy() - o).max(), ctx.stats())
        if not np.array_equal(sg, so):
            print(" gpu[:20]", sg[:20], "\n orc[:20]", so[:20])
    ctx.close()
