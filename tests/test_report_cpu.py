"""Measured report bundle (report.py): calibration, modeled-vs-measured table,
ladder and transition bookkeeping -- host logic over the control plane."""
import json
import os

from paper_2102_03161_b200 import LIB_PATH, configs, report
from paper_2102_03161_b200.capi import EpsApi
from paper_2102_03161_b200.trainer import EpochResult, Trainer

API = EpsApi(LIB_PATH, "eps_")


def _rows_from_model(scen, scale=1.0, trans=0.0):
    rows, _ = report.modeled(API, scen)
    return [EpochResult(r["epoch"], r["l_frozen"], r["pipeline_length"], r["replica_width"],
                        r["micro_batches"], r["iteration_time"] * scale,
                        r["epoch_time"] * scale, r["throughput"] / scale, bool(r["cache_enabled"]),
                        False, trans if i else 0.0, 1.0)
            for i, r in enumerate(rows)]


def test_calibration_recovers_scaled_forward_rate():
    scen = configs.scenario("vit-b16", 1)
    rows, _ = report.modeled(API, scen)
    target = rows[0]["iteration_time"] * 0.1  # a 10x faster device
    cal = report.calibrate_c_fwd(API, scen, target)
    assert abs(cal["modeled_iteration_s"] - target) <= 1e-6 * target
    assert cal["c_fwd"] < scen["cost_model"]["c_fwd"]
    # the calibrated scenario keeps every other field
    s = dict(cal["scenario"])
    s["cost_model"] = dict(s["cost_model"], c_fwd=scen["cost_model"]["c_fwd"])
    assert s == scen


def test_compare_and_transitions():
    scen = configs.scenario("vit-b16", 8)
    meas = _rows_from_model(scen, scale=0.5, trans=0.25)
    rows, _ = report.modeled(API, scen)
    cmp = report.compare(rows, meas)
    assert all(c["decisions_match"] for c in cmp)
    assert all(abs(c["measured_over_modeled"] - 0.5) < 1e-9 for c in cmp)
    tt = report.transition_table(scen, meas)
    ks = [r["pipeline_length"] for r in rows]
    assert len(tt) == sum(1 for a, b in zip(ks, ks[1:]) if a != b) > 0
    assert all(t["measured_s"] == 0.25 for t in tt)


def test_ladder_and_bundle(tmp_path):
    scen = configs.scenario("vit-b16", 1)
    seen = []

    def fake_rung(s):
        seen.append(s["features"])
        return 10.0 if not s["features"]["freeze"] else 5.0

    lad = report.ladder(API, scen, fake_rung)
    assert [r["rung"] for r in lad] == ["baseline", "freeze", "all"]
    assert lad[0]["measured_speedup"] == 1.0 and lad[2]["measured_speedup"] == 2.0
    assert seen[0] == {"freeze": False, "autopipe": False, "autodp": False, "autocache": False}
    meas = _rows_from_model(scen)
    tl = [{"device": 0, "kind": "F", "start_s": 0.0, "end_s": 0.01, "tag": "mb0"}]
    files = report.bundle(str(tmp_path), API, scen, meas, tl, lad)
    assert set(files) >= {"epochs.csv", "timeline.json", "modeled_vs_measured.json",
                          "calibrated_scenario.json", "ladder.json"}
    csv = open(files["epochs.csv"]).read().splitlines()
    assert csv[0] == Trainer.report_csv([]).splitlines()[0] and len(csv) == len(meas) + 1
    mvm = json.load(open(files["modeled_vs_measured.json"]))
    assert mvm["calibrated"]["c_fwd"] > 0
    assert all(e["decisions_match"] for e in mvm["calibrated"]["epochs"])
    assert os.path.exists(files["timeline.json"])


def test_alpha_sweep_is_monotone_in_the_model():
    scen = configs.scenario("vit-b16", 1)
    rows = report.alpha_sweep(API, scen, lambda s: 1.0 / (1.0 + s["training"]["alpha"]),
                              alphas=(0.2, 0.5), baseline_total_s=1.0)
    assert [r["alpha"] for r in rows] == [0.2, 0.5]
    assert rows[1]["modeled_speedup"] >= rows[0]["modeled_speedup"]
    assert sum(rows[1]["frozen_trajectory"]) >= sum(rows[0]["frozen_trajectory"])


def test_chunks_sweep_model_matches_reference_choice():
    """The sweep's modeled side is the reference's optimal_chunks: at 1x8 the
    epoch-0 choice is M = 23 (SURVEY.md 8(a) a7 golden), and the measured
    slope over M is recovered (the per-micro-batch overhead)."""
    scen = configs.scenario("vit-b16", 8)
    rows = report.chunks_sweep(API, scen, 8, lambda m: 0.25 + 0.002 * m)
    assert [r["m"] for r in rows] == list(range(8, 49))
    assert [r["m"] for r in rows if r["is_optimal"]] == [23]
    assert abs(rows[0]["measured_per_microbatch_s"] - 0.002) < 1e-12
    one = report.chunks_sweep(API, configs.scenario("vit-b16", 1), 1, lambda m: 0.04,
                              calibrated_c_fwd=1e-13)
    assert [r["m"] for r in one] == [1, 2, 3, 4, 5, 6]
    assert all(r["calibrated_modeled_iteration_s"] < r["modeled_iteration_s"] for r in one)


def test_chunks_sweep_custom_model_spec():
    """Scenarios with explicit model arrays (tiny ViT, BERT, CIFAR ViT: no
    preset) go through the same sweep (tools/multi_gpu_sweeps.py uses them)."""
    for cfg in ("tiny-vit", "bert-large-128"):
        scen = configs.scenario(cfg, 2)
        assert "preset" not in scen["model"]
        rows = report.chunks_sweep(API, scen, 2, lambda m: 0.01 + 0.001 * m)
        assert [r["m"] for r in rows] == list(range(2, 13))
        assert sum(r["is_optimal"] for r in rows) == 1
        assert all(r["modeled_iteration_s"] > 0 for r in rows)


def test_bandwidth_sweep_comm_ratio_falls_with_bandwidth():
    scen = configs.scenario("vit-b16", 8)
    scen["cluster"]["nodes"] = 2  # 2 x 8: the replicas' all-reduce crosses nodes
    rows = report.bandwidth_sweep(API, scen, [1e9, 5e9, 25e9], calibrated_c_fwd=1e-12)
    assert [r["inter_node_bandwidth"] for r in rows] == [1e9, 5e9, 25e9]
    assert rows[0]["comm_ratio"] > rows[1]["comm_ratio"] > rows[2]["comm_ratio"]
    assert rows[0]["total_time_s"] > rows[2]["total_time_s"]
    # a faster device makes communication a larger share of the iteration
    assert all(r["calibrated_comm_ratio"] >= r["comm_ratio"] for r in rows)
