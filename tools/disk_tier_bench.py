"""AutoCache disk tier on ViT-B/16 b400: gather-epoch
iteration time reading the cached boundary activations from a file through
the DiskTier host window, beside the HBM tier, with the measured stall next
to the reference's modeled one (CacheTierSim, autocache.cpp:69-150, driven as
runner.cpp:258-265 with the measured read bandwidth and the HBM tier's
iteration time).

    python tools/disk_tier_bench.py [iters] [window_batches] [block_batches] [dir]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_03161_b200 import LIB_PATH, configs  # noqa: E402
from paper_2102_03161_b200.capi import CacheTierParams, EpsApi  # noqa: E402
from paper_2102_03161_b200.trainer import Trainer  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 8
wb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
bb = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cache_dir = sys.argv[4] if len(sys.argv) > 4 else None
epochs = 8
scen = configs.scenario("vit-b16", 1)
scen["cache"]["window_batches"] = wb
scen["cache"]["block_batches"] = bb
g = configs.GEOMETRIES["vit-b16"]
out = {"iters_per_epoch": iters, "window_batches": wb, "block_batches": bb, "epochs": {}}
gather_ms = {}
for tier in ("hbm", "disk"):
    tr = Trainer(scen, g, iterations_per_epoch=iters, device_norms=False, cache_tier=tier,
                 cache_dir=cache_dir)
    rows = tr.run(epochs)
    out["epochs"][tier] = [{"epoch": r.epoch, "l_frozen": r.l_frozen,
                            "cache": "move" if r.cache_moved else (
                                "gather" if r.cache_enabled else "off"),
                            "ms_per_iteration": round(r.iteration_time_s * 1e3, 3),
                            "stall_s": round(r.stall_time_s, 4)} for r in rows]
    gather_ms[tier] = [r.iteration_time_s * 1e3 for r in rows
                       if r.cache_enabled and not r.cache_moved]
    if tier == "disk":
        out["disk_stats"] = tr.disk_stats
        row_bytes = g.tokens * g.hidden * 2
    del tr
api = EpsApi(LIB_PATH, "eps_")
gathers = [s for s in out["disk_stats"] if s["mode"] == 1]
if gathers:
    s1 = gathers[-1]
    rd = s1["bytes_read"] - (gathers[-2]["bytes_read"] if len(gathers) > 1 else 0.0)
    busy = s1["read_busy_s"] - (gathers[-2]["read_busy_s"] if len(gathers) > 1 else 0.0)
    per_thread_bw = rd / busy if busy > 0 else float("nan")
    it_s = min(gather_ms["hbm"]) / 1e3
    bpb = row_bytes * configs.BATCH["vit-b16"]
    t = CacheTierParams(disk_bandwidth=per_thread_bw, window_batches=wb, block_batches=bb)
    out["model"] = {"disk_bandwidth_per_thread_Bps": per_thread_bw,
                    "hbm_tier_iteration_s": it_s,
                    "cache_tier_sim": api.cache_tier_epoch(t, bpb, iters, it_s),
                    "note": "CacheTierSim fetches one block at a time; the disk tier runs "
                            "8 reader threads, so the measured stall can undercut the model"}
    out["measured_gather_stall_s"] = [r["stall_s"] for r in out["epochs"]["disk"]
                                      if r["cache"] == "gather"]
out["gather_ms_per_iteration"] = {k: [round(x, 3) for x in v] for k, v in gather_ms.items()}
print(json.dumps(out))
