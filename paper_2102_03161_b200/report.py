"""Measured report bundle.

The reference *models* every epoch (runner.cpp:94-305) and writes a CSV
(runner.cpp:340-355), a timeline (runner.cpp:357-367) and a feature ladder
(speedup_breakdown, runner.cpp:307-338) from its cost model.  This module puts
the *measured* B200 numbers beside the modeled ones:

* `calibrate_c_fwd`: fit the cost model's forward rate `c_fwd`
  (cost_model.hpp:12, seconds per parameter-sample) so the modeled epoch-0
  iteration equals the measured one -- the reference's constants describe RTX
  5000s; a calibrated scenario replays the planner with B200 costs;
* `compare`: per-epoch modeled vs measured iteration time (same decisions);
* `ladder`: measured rungs of the feature ladder next to the modeled ones;
* `alpha_sweep`: the freeze-aggressiveness sweep (cli.cpp:75-135) measured;
* `chunks_sweep`: the micro-batch-count sweep (cli.cpp:96-117) measured;
* `bandwidth_sweep`: the interconnect sweep (cli.cpp:118-127), modeled with the reference's
  and with the B200-calibrated constants;
* `bundle`: writes epochs.csv (reference schema, measured), timeline.json
  (reference schema, measured CUDA-event blocks), calibration / comparison /
  ladder JSON.

Transition overheads (8(f) row 4) are measured by Trainer.run_epoch (CUDA
events around StageRunner.set_plan: migration + regroup + store hand-over) and
land in the CSV's transition_overhead_s column; `transition_table` lists them
next to the reference's Table-3 constants (runner.cpp:24-28).
"""
from __future__ import annotations

import copy
import json
import math
import os
from typing import Callable, Dict, List, Sequence

from .capi import EpsApi, Scenario

# The feature-ladder rungs of runner.cpp:312-319 (freeze, autopipe, autodp, autocache).
LADDER = [
    ("baseline", (False, False, False, False)),
    ("freeze", (True, False, False, False)),
    ("autopipe", (True, True, False, False)),
    ("autopipe+autocache", (True, True, False, True)),
    ("autopipe+autodp", (True, True, True, False)),
    ("all", (True, True, True, True)),
]


def with_features(scenario: dict, flags: Sequence[bool]) -> dict:
    s = copy.deepcopy(scenario)
    s["features"] = dict(zip(("freeze", "autopipe", "autodp", "autocache"), map(bool, flags)))
    return s


def modeled(api: EpsApi, scenario: dict):
    """The reference's modeled run (simulate_run): per-epoch rows + summary."""
    return Scenario(api, scenario).simulate()


def calibrate_c_fwd(api: EpsApi, scenario: dict, measured_iteration_s: float,
                    epoch: int = 0, iters: int = 60) -> dict:
    """Bisect (in log space) the cost model's c_fwd so the modeled iteration
    time of `epoch` equals `measured_iteration_s`.  The modeled time is
    monotone in c_fwd (every F/B block scales with it; comm and per-micro-batch
    overheads do not).  Returns {c_fwd, modeled_iteration_s, scenario}."""
    if measured_iteration_s <= 0:
        raise ValueError("measured iteration time must be positive")

    def t_of(c):
        s = copy.deepcopy(scenario)
        s["cost_model"]["c_fwd"] = c
        rows, _ = modeled(api, s)
        return rows[epoch]["iteration_time"], s

    lo, hi = 1e-18, 1e-6
    t_lo, _ = t_of(lo)
    if t_lo >= measured_iteration_s:  # overheads alone exceed the measurement
        return {"c_fwd": lo, "modeled_iteration_s": t_lo, "scenario": t_of(lo)[1],
                "note": "fixed overheads exceed the measured iteration"}
    for _ in range(iters):
        mid = math.sqrt(lo * hi)
        t, _ = t_of(mid)
        if t < measured_iteration_s:
            lo = mid
        else:
            hi = mid
    c = math.sqrt(lo * hi)
    t, s = t_of(c)
    return {"c_fwd": c, "modeled_iteration_s": t, "scenario": s}


def compare(modeled_rows: List[dict], measured_rows) -> List[dict]:
    """Epoch-by-epoch: decisions must agree; iteration times side by side."""
    out = []
    for m, r in zip(modeled_rows, measured_rows):
        same = (m["l_frozen"], m["pipeline_length"], m["replica_width"], m["micro_batches"]) == (
            r.l_frozen, r.k, r.r, r.m)
        out.append({"epoch": r.epoch, "l_frozen": r.l_frozen, "k": r.k, "r": r.r, "m": r.m,
                    "decisions_match": same,
                    "modeled_iteration_s": m["iteration_time"],
                    "measured_iteration_s": r.iteration_time_s,
                    "measured_over_modeled": r.iteration_time_s / m["iteration_time"]
                    if m["iteration_time"] > 0 else None,
                    "modeled_transition_s": m["transition_overhead"],
                    "measured_transition_s": r.transition_time_s})
    return out


def ladder(api: EpsApi, scenario: dict, run_rung: Callable[[dict], float],
           rungs: Sequence[str] = ("baseline", "freeze", "all")) -> List[dict]:
    """Measured total time of each rung (run_rung(scenario) -> seconds) with
    speedups vs the measured baseline, beside the reference's modeled ladder."""
    model = {name: (t, sps, sp) for name, t, sps, sp in Scenario(api, scenario).speedup_breakdown()}
    flags = dict(LADDER)
    out, base = [], None
    for name in rungs:
        t = run_rung(with_features(scenario, flags[name]))
        base = t if name == "baseline" else base
        out.append({"rung": name, "measured_total_s": t,
                    "measured_speedup": (base / t) if base else None,
                    "modeled_total_s": model[name][0], "modeled_speedup": model[name][2]})
    return out


def alpha_sweep(api: EpsApi, scenario: dict, run_total: Callable[[dict], float],
                alphas: Sequence[float] = (0.2, 1.0 / 3.0, 0.4, 0.5),
                baseline_total_s: float = None) -> List[dict]:
    """The freeze-aggressiveness sweep of cli.cpp:75-135 (Eq. 1's alpha) run on
    the device: measured total time and speedup vs the no-freeze baseline per
    alpha, beside the modeled speedup and the frozen-layer trajectory."""
    base = baseline_total_s if baseline_total_s is not None else run_total(
        with_features(scenario, dict(LADDER)["baseline"]))
    out = []
    for a in alphas:
        s = copy.deepcopy(scenario)
        s["training"]["alpha"] = a
        rows, summ = modeled(api, s)
        t = run_total(s)
        out.append({"alpha": a, "frozen_trajectory": [r["l_frozen"] for r in rows],
                    "measured_total_s": t, "measured_speedup": base / t,
                    "modeled_speedup": summ["speedup"]})
    return out


def chunks_sweep(api: EpsApi, scenario: dict, k: int, run_m: Callable[[int], float],
                 calibrated_c_fwd: float = None) -> List[dict]:
    """The chunks sweep of cli.cpp:96-117 on the device: for pipeline length
    `k` (L_f = 0 plan from load_balance, replica width from the topology) the
    reference's modeled iteration time for every M in [k, 6k] (optimal_chunks,
    chunks.cpp:5-24) beside the measured one (run_m(M) -> seconds per
    iteration).  With `calibrated_c_fwd` the model is also replayed with the
    B200-calibrated forward rate.  The measured slope over M is the device's
    per-micro-batch overhead (cost_model per_microbatch_overhead)."""
    from .capi import ClusterSpec, CostModel

    cl_d, cm_d = scenario["cluster"], scenario["cost_model"]
    cluster = ClusterSpec(cl_d["nodes"], cl_d["gpus_per_node"], cl_d["gpu_memory_bytes"],
                          cl_d["intra_node_bandwidth"], cl_d["inter_node_bandwidth"])
    cost = CostModel(cm_d["c_fwd"], cm_d["backward_ratio"], cm_d["c_update"],
                     cm_d["per_microbatch_overhead"], cm_d["allreduce_bucket_bytes"],
                     cm_d["comm_latency"])
    md = scenario["model"]
    if "preset" in md:
        model = api.model_preset(md["preset"])
    else:  # explicit arrays (configs.scenario for the tiny ViT / BERT / CIFAR configs)
        from .capi import ModelSpec
        model = ModelSpec(list(md["attention_params"]), list(md["mlp_params"]),
                          list(md["activation_bytes"]), int(md.get("bytes_per_param", 4)),
                          md.get("name", "custom"))
    seq = api.m_partition(model, 0)
    crit = 1 if scenario.get("balance_criterion") == "paper-variance" else 0  # scenario.cpp:219-225
    plan = api.load_balance(seq, k, scenario["training"]["lambda_frozen"], crit)
    _, r = api.topology(cluster, k)
    batch = float(scenario["training"]["per_pipeline_batch"])
    chosen, times = api.optimal_chunks(plan, model, seq, batch, r, cluster, cost)
    cal_times = None
    if calibrated_c_fwd is not None:
        cost_cal = CostModel(**{**cost.__dict__, "c_fwd": calibrated_c_fwd})
        _, cal_times = api.optimal_chunks(plan, model, seq, batch, r, cluster, cost_cal)
    out = []
    for i, m in enumerate(range(k, 6 * k + 1)):
        row = {"k": k, "m": m, "modeled_iteration_s": times[i], "is_optimal": m == chosen,
               "measured_iteration_s": run_m(m)}
        if cal_times is not None:
            row["calibrated_modeled_iteration_s"] = cal_times[i]
        out.append(row)
    if len(out) > 1:  # least-squares slope of measured time over M
        ms = [o["m"] for o in out]
        ts = [o["measured_iteration_s"] for o in out]
        mb, tb = sum(ms) / len(ms), sum(ts) / len(ts)
        slope = sum((a - mb) * (b - tb) for a, b in zip(ms, ts)) / sum((a - mb) ** 2 for a in ms)
        for o in out:
            o["measured_per_microbatch_s"] = slope
    return out


def bandwidth_sweep(api: EpsApi, scenario: dict, values: Sequence[float],
                    calibrated_c_fwd: float = None) -> List[dict]:
    """The bandwidth sweep of cli.cpp:118-127: the modeled run per
    inter-node bandwidth (comm ratio, speedup, total time), with the
    reference's constants and, given `calibrated_c_fwd`, with the B200
    forward rate -- the calibrated model is what a multi-node B200 run is
    predicted to see (one GPU cannot vary its interconnect)."""
    out = []
    for bw in values:
        s = copy.deepcopy(scenario)
        s["cluster"]["inter_node_bandwidth"] = float(bw)
        _, summ = modeled(api, s)
        row = {"inter_node_bandwidth": float(bw), "comm_ratio": summ["comm_ratio"],
               "speedup": summ["speedup"], "total_time_s": summ["total_seconds"]}
        if calibrated_c_fwd is not None:
            s["cost_model"]["c_fwd"] = calibrated_c_fwd
            _, sc = modeled(api, s)
            row.update(calibrated_comm_ratio=sc["comm_ratio"], calibrated_speedup=sc["speedup"],
                       calibrated_total_time_s=sc["total_seconds"])
        out.append(row)
    return out


def transition_table(scenario: dict, measured_rows) -> List[dict]:
    """Measured plan-change overheads beside the scenario's Table-3 constants."""
    consts = scenario.get("cost_model", {}).get("transition_overheads", {})
    out, prev_k = [], None
    for r in measured_rows:
        if prev_k is not None and r.k != prev_k:
            key = f"{prev_k}->{r.k}"
            out.append({"epoch": r.epoch, "transition": key,
                        "measured_s": r.transition_time_s, "reference_constant_s": consts.get(key)})
        prev_k = r.k
    return out


def bundle(out_dir: str, api: EpsApi, scenario: dict, measured_rows, timeline: List[dict],
           ladder_rows: List[dict] = None, extra: Dict = None,
           sweep_rows: List[dict] = None, chunks_rows: List[dict] = None) -> Dict[str, str]:
    """Write the measured report bundle; returns {name: path}."""
    from .trainer import Trainer  # local: trainer imports torch

    os.makedirs(out_dir, exist_ok=True)
    rows_mod, summ = modeled(api, scenario)
    cal = calibrate_c_fwd(api, scenario, measured_rows[0].iteration_time_s)
    rows_cal, summ_cal = modeled(api, cal["scenario"])
    files = {}

    def dump(name, obj):
        path = os.path.join(out_dir, name)
        with open(path, "w") as f:
            if isinstance(obj, str):
                f.write(obj)
            else:
                json.dump(obj, f, indent=1)
        files[name] = path

    dump("epochs.csv", Trainer.report_csv(measured_rows))
    dump("timeline.json", timeline)
    measured_total = sum(r.epoch_time_s + r.transition_time_s for r in measured_rows)
    dump("modeled_vs_measured.json", {
        "reference_constants": {"epochs": compare(rows_mod, measured_rows),
                                "modeled_total_s": summ["total_seconds"],
                                "modeled_speedup": summ["speedup"]},
        "calibrated": {"c_fwd": cal["c_fwd"],
                       "reference_c_fwd": scenario["cost_model"]["c_fwd"],
                       "epochs": compare(rows_cal, measured_rows),
                       "modeled_total_s": summ_cal["total_seconds"],
                       "modeled_speedup": summ_cal["speedup"]},
        "measured_total_s": measured_total,
        "transitions": transition_table(scenario, measured_rows),
        **(extra or {})})
    dump("calibrated_scenario.json", cal["scenario"])
    if ladder_rows is not None:
        dump("ladder.json", ladder_rows)
    if sweep_rows is not None:
        dump("alpha_sweep.json", sweep_rows)
    if chunks_rows is not None:
        dump("chunks_sweep.json", chunks_rows)
    return files
