"""Host-tier AutoCache on ViT-B/16 b400: gather-epoch iteration time with the
prefetch window (copy-stream gathers one iteration ahead) vs direct host
gathers vs the HBM tier.

    python tools/host_tier_bench.py [epochs] [iters]      (on a B200)
"""
import json
import sys

sys.path.insert(0, ".")
from paper_2102_03161_b200 import configs  # noqa: E402
from paper_2102_03161_b200.trainer import Trainer  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
scen = configs.scenario("vit-b16", 1)
g = configs.GEOMETRIES["vit-b16"]
out = {}
variants = {"hbm": (dict(cache_tier="hbm"), 0),
            "host_direct": (dict(cache_tier="host", cache_prefetch=False), 0)}
for ctas in (8, 16, 32):
    variants[f"host_window_{ctas}"] = (dict(cache_tier="host", cache_prefetch=True), ctas)
for name, (kw, ctas) in variants.items():
    tr = Trainer(scen, g, iterations_per_epoch=iters, device_norms=False, **kw)
    if ctas:
        tr.cache_prefetch_ctas = ctas
    rows = tr.run(epochs)
    out[name] = [{"epoch": r.epoch, "l_frozen": r.l_frozen,
                  "cache": "move" if r.cache_moved else ("gather" if r.cache_enabled else "off"),
                  "ms_per_iteration": round(r.iteration_time_s * 1e3, 3)} for r in rows]
    del tr
for name, rows in out.items():
    g_ms = [r["ms_per_iteration"] for r in rows if r["cache"] == "gather"]
    print(json.dumps({"tier": name, "gather_epoch_ms_per_iteration": g_ms, "epochs": rows}))
