"""Measured report bundle on one B200.

Runs the reference's vit-b16 scenario (BASELINE config 2, G=1) through the
real epoch loop with the scenario's own norm source (so every decision equals
the modeled one), then writes gpurun_out/<tag>_report/ (copied to profiles/): epochs.csv (reference
schema, measured), timeline.json (measured F/B blocks of the last iteration),
modeled_vs_measured.json (reference constants and B200-calibrated c_fwd),
calibrated_scenario.json, ladder.json (baseline / freeze / all, measured
beside the modeled ladder) and alpha_sweep.json (Eq. 1's alpha, measured).

    python tools/measured_report.py [tag] [iterations_per_epoch]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2102_03161_b200 import LIB_PATH, configs, report  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.trainer import Trainer  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01e"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "gpurun_out", f"{tag}_report")
api = EpsApi(LIB_PATH, "eps_")
geom = configs.GEOMETRIES["vit-b16"]
scen = configs.scenario("vit-b16", 1)
scen["training"]["iterations_per_epoch"] = iters


def run(s, trace=False):
    tr = Trainer(s, geom, iterations_per_epoch=iters, device_norms=False)
    tr.run_epoch(0)  # warm-up epoch (kernels configured, allocator primed)
    tr = Trainer(s, geom, iterations_per_epoch=iters, device_norms=False)
    if trace:
        tr.runner.trace = []
    rows = tr.run()
    torch.cuda.synchronize()
    return tr, rows


tr, rows = run(scen, trace=True)
timeline = tr.runner.timeline()
del tr
torch.cuda.empty_cache()


def rung(s):
    t, r = run(s)
    del t
    torch.cuda.empty_cache()
    return sum(x.epoch_time_s + x.transition_time_s for x in r)


lad = report.ladder(api, scen, rung)
sweep = report.alpha_sweep(api, scen, rung, baseline_total_s=lad[0]["measured_total_s"])
files = report.bundle(out, api, scen, rows, timeline, lad, sweep_rows=sweep,
                      extra={"device": torch.cuda.get_device_name(),
                             "iterations_per_epoch": iters,
                             "note": "measured epochs run `iterations_per_epoch` iterations; "
                                     "per-iteration times compare directly with the model"})
print(json.dumps({k: os.path.relpath(v) for k, v in files.items()}))
print(json.dumps(lad))
print(json.dumps(sweep))
