"""Print the key numbers of bench JSON lines (usage: python tools/show_bench.py file.json ...)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e)
        continue
    print("=====", f, d["config"]["workload"][:3], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4),
          "e2e", round(d["e2e"]["value"], 1), "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    for k in ("roofline", "roofline_layer_hbm", "roofline_full_cache", "roofline_kmeans"):
        r = d.get(k)
        if r:
            print(f"  {k:20s} {r['kernel'][:24]:24s} ach {r['achieved']:.1f} / {r['peak']:.0f} {r['unit']} frac "
                  f"{r['frac']:.3f} share {r.get('share_of_step') or 0:.3f} ms/launch {r.get('ms_per_launch')}")
    lu = d["layer_us"]
    print("  layer_us unflagged %.2f flagged %.2f full %.2f  ret/layer-step %.4f" % (
        lu["retrieval_unflagged"], lu["retrieval_flagged"], lu["full_cache"], d["retrievals_per_layer_step"]))
    km = d["kmeans"]
    print("  kmeans keys/s %.3g non-gemm %.3f phases %s" % (km["keys_per_s_lloyd"], km["non_gemm_share_of_iteration"],
                                                            {k: round(v, 2) for k, v in km["phase_ms"].items()}))
    if d.get("l2_pressure"):
        print("  l2", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in d["l2_pressure"].items() if k != "note"})
