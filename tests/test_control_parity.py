"""Bit-exact parity of the product control plane (libeps_b200.so) with the
reference's own implementation.

Two oracles:
  * committed golden fixtures produced by the reference (tests/golden/), so
    these tests run anywhere;
  * the reference compiled from its sources (oracle/_ref/libeps_ref.so,
    built by `make oracle`), driven through the very same C ABI for
    randomised call-for-call comparison.
"""
import json
import math
import os

import pytest

from paper_2102_03161_b200 import LIB_PATH, configs
from paper_2102_03161_b200.capi import (ClusterSpec, CostModel, CacheTierParams, DomainError,
                                        EpsApi, InvalidArgument, SublayerSeq)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle/_ref/libeps_ref.so")
GOLDEN = json.load(open(os.path.join(ROOT, "tests/golden/decisions.json")))


@pytest.fixture(scope="module")
def prod():
    return EpsApi(LIB_PATH, "eps_")


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (make oracle)")
    return EpsApi(REF_LIB, "epsref_")


@pytest.mark.parametrize("case", GOLDEN["scenarios"], ids=lambda c: c["name"])
def test_simulate_run_matches_golden(prod, case):
    s = prod.scenario(case["scenario"])
    rows, summ = s.simulate()
    assert rows == case["rows"]  # every field, doubles included, bit for bit
    for k, v in case["summary"].items():
        assert summ[k] == v, k
    assert s.report(0) == case["report_csv"]
    assert s.report(3) == case["transitions_jsonl"]
    if case["breakdown"] is not None:
        assert [list(r) for r in s.speedup_breakdown()] == case["breakdown"]


@pytest.mark.parametrize("case", GOLDEN["scenarios"], ids=lambda c: c["name"])
def test_epoch_planner_replays_decisions(prod, case):
    """The training loop's EpochPlanner takes the same decisions as simulate_run."""
    from paper_2102_03161_b200.planner import Planner
    p = Planner(prod, case["scenario"])
    for row in case["rows"]:
        d = p.begin_epoch(row["epoch"])
        assert (d.l_frozen, d.pipeline_length, d.replica_width, d.micro_batches,
                int(d.cache_enabled)) == (row["l_frozen"], row["pipeline_length"],
                                          row["replica_width"], row["micro_batches"],
                                          row["cache_enabled"])


def test_scenario_round_trip(prod, ref):
    for case in GOLDEN["scenarios"][:6]:
        a = prod.scenario(case["scenario"]).to_json()
        b = ref.scenario(case["scenario"]).to_json()
        assert a == b
        assert prod.scenario(a).to_json() == a


@pytest.mark.parametrize("bad,err", [
    ({"schema_version": 1, "model": {"preset": "vit-b16"}, "bogus": 1}, "unknown key"),
    ({"schema_version": 2, "model": {"preset": "vit-b16"}}, "schema_version"),
    ({"schema_version": 1}, "model is required"),
    ({"schema_version": 1, "model": {"preset": "vit-b16"}, "cluster": {"nodes": "x"}},
     "wrong type"),
    ({"schema_version": 1, "model": {"preset": "vit-b16"},
      "features": {"freeze": False, "autopipe": True}}, "autopipe requires freeze"),
])
def test_scenario_strictness(prod, ref, bad, err):
    from paper_2102_03161_b200.capi import ConfigError
    for api in (prod, ref):
        with pytest.raises(ConfigError, match=err):
            api.scenario(bad)


def _rng(seed):
    import random
    return random.Random(seed)


def test_load_balance_and_compress_random(prod, ref):
    r = _rng(2024)
    for trial in range(600):
        k = r.choice([1, 2, 4, 8])
        n = k + r.randrange(0, 48 - k + 1)
        sizes = [1 + r.randrange(1_000_000_000) for _ in range(n)]
        if trial % 3 == 0:  # transformer-like stacks with exact ties
            sizes = [r.choice([2_363_904, 4_723_968, 4_200_448]) for _ in range(n)]
        fl = r.randrange(0, 6)
        seq = SublayerSeq(sizes, [2 * fl + i for i in range(n)],
                          r.randrange(0, 10_000_000_000), fl)
        lam = r.random() if trial % 2 else 1 / 6
        crit = trial % 5 == 0
        a = prod.load_balance(seq, k, lam, int(crit))
        b = ref.load_balance(seq, k, lam, int(crit))
        assert a == b
        m0 = a.max_effective_size() * r.choice([0.5, 1.0, 2.0, 10.0])
        assert prod.try_compress(seq, k, lam, m0, int(crit)) == ref.try_compress(seq, k, lam, m0,
                                                                                 int(crit))


def test_load_balance_errors(prod, ref):
    seq = SublayerSeq([1, 2, 3], [0, 1, 2])
    for api in (prod, ref):
        with pytest.raises(InvalidArgument):
            api.load_balance(seq, 4, 0.0)
        with pytest.raises(InvalidArgument):
            api.try_compress(SublayerSeq([1, 2, 3, 4, 5, 6], list(range(6))), 3, 0.0, 100.0)


def test_optimal_chunks_random(prod, ref):
    r = _rng(7)
    model = prod.model_preset("vit-b16")
    assert model == ref.model_preset("vit-b16")
    for trial in range(120):
        lf = r.randrange(0, 12)
        seq = prod.m_partition(model, lf)
        assert seq == ref.m_partition(model, lf)
        k = r.choice([kk for kk in (1, 2, 4, 8) if kk <= len(seq.params)])
        plan = prod.load_balance(seq, k, 1 / 6)
        cl = ClusterSpec(r.choice([1, 2]), 8, 16e9, r.choice([15.754e9, 9e11]), 12e9)
        cm = CostModel(c_fwd=r.choice([9.722222222222221e-12, 1e-9]),
                       per_microbatch_overhead=r.choice([0.0, 2e-4, 8e-4]),
                       comm_latency=r.choice([0.0, 1e-5]))
        R = r.choice([1, 2, 4, 8])
        batch = r.choice([64.0, 320.0, 400.0, 37.0])
        cache = trial % 2 == 0
        read = r.random() * 1e-4
        assert prod.optimal_chunks(plan, model, seq, batch, R, cl, cm, cache, read) == \
            ref.optimal_chunks(plan, model, seq, batch, R, cl, cm, cache, read)


def test_build_schedule_random(prod, ref):
    r = _rng(11)
    for trial in range(200):
        k = r.choice([1, 2, 3, 4, 8])
        stages = [(r.choice([0.0, r.random() * 1e7]), r.choice([0.0, r.random() * 1e7]),
                   r.random() * 1e-3, r.random() * 1e6) for _ in range(k)]
        m = r.randrange(1, 6 * k + 1)
        cm = CostModel(c_fwd=1e-9, c_update=2e-10, per_microbatch_overhead=1e-4,
                       allreduce_bucket_bytes=r.choice([1e6, 25e6]),
                       comm_latency=r.choice([0.0, 1e-5]))
        kw = dict(integer_microbatches=trial % 2 == 0, group_spans_nodes=trial % 3 == 0,
                  intra=1e12, inter=1e10, cm=cm)
        for width in (1, 4):
            assert prod.build_schedule(stages, m, 128.0, width, **kw) == \
                ref.build_schedule(stages, m, 128.0, width, **kw)


def test_freeze_trajectories_random(prod, ref):
    r = _rng(99)
    for trial in range(60):
        alpha = 0.1 + 0.8 * r.random()
        L = r.choice([4, 12, 24])
        fp, fr = prod.freeze_state(alpha), ref.freeze_state(alpha)
        for t in range(20):
            norms = [r.random() for _ in range(L)]
            if t % 4 == 0:
                norms = [1.0] * L
            assert fp.next(norms) == fr.next(norms)
    for profile in (0, 1):
        for seed in (0, 5, 17, 42):
            for L in (4, 12, 24):
                for e in range(8):
                    assert prod.synthetic_norms(profile, seed, L, 2, e) == \
                        ref.synthetic_norms(profile, seed, L, 2, e)
    for t in range(1, 30):
        assert prod.frozen_bound_closed_form(t, 12, 0.3) == ref.frozen_bound_closed_form(t, 12, 0.3)


def test_freeze_errors(prod, ref):
    for api in (prod, ref):
        st = api.freeze_state(0.5)
        with pytest.raises(DomainError):
            st.next([1.0] * 10, 12)
        with pytest.raises(DomainError):
            st.next([1.0, -1.0, 1.0])
        with pytest.raises(DomainError):
            api.freeze_state(1.0)


def test_trace_source(prod, ref, tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("epoch,layer,grad_norm\n" + "".join(
        f"{e},{l},{10.0 * e + l + 0.5}\n" for e in range(2) for l in range(3)))
    for api in (prod, ref):
        assert api.trace_norms(str(p), 1) == [10.5, 11.5, 12.5]
        with pytest.raises(DomainError):
            api.trace_norms(str(p), 2)
    p.write_text("epoch,layer,grad_norm\n0,0,1.0\n0,2,1.0\n")
    for api in (prod, ref):
        with pytest.raises(DomainError):
            api.trace_norms(str(p), 0)


def test_autodp_random(prod, ref):
    r = _rng(5)
    for nodes in (1, 2):
        for gpn in (1, 2, 4, 8):
            ks = [k for k in (1, 2, 4, 8) if gpn % k == 0]
            for k in ks:
                cl = ClusterSpec(nodes, gpn)
                assert prod.topology(cl, k) == ref.topology(cl, k)
                for nk in ks:
                    if nk <= k:
                        assert prod.transition(cl, k, nk, 3, 0.3, 6, "v3") == \
                            ref.transition(cl, k, nk, 3, 0.3, 6, "v3")
                for _ in range(3):
                    ds = r.randrange(nodes * gpn, 3000)
                    e, seed = r.randrange(10), r.randrange(1 << 63)
                    assert prod.redistribute(ds, cl, k, e, seed) == \
                        ref.redistribute(ds, cl, k, e, seed)
    with pytest.raises(DomainError):
        prod.transition(ClusterSpec(2, 8), 4, 8)
    with pytest.raises(DomainError):
        prod.redistribute(7, ClusterSpec(2, 8), 2, 0, 1)


def test_autocache_random(prod, ref):
    model = prod.model_preset("vit-b16")
    r = _rng(3)
    for _ in range(200):
        t = CacheTierParams(host_bandwidth=r.choice([3.05e9, 1e12, 3e13]),
                            read_latency=r.choice([0.0, 1e-6]))
        cm = CostModel(c_fwd=r.choice([9.722222222222221e-12, 1e-13]))
        lf = r.randrange(0, 13)
        mb = r.choice([1.0, 17.4, 400.0])
        assert prod.should_cache(lf, model, cm, t, mb) == ref.should_cache(lf, model, cm, t, mb)
        old = r.randrange(0, 12)
        new = r.randrange(old, 13)
        assert prod.cache_transition(True, old, t, old, new, model, cm) == \
            ref.cache_transition(True, old, t, old, new, model, cm)


def test_cache_tier_epoch_random(prod, ref):
    """The modeled disk -> host window (CacheTierSim, the model the disk tier's
    measured stalls are reported beside) equals the reference call for call."""
    r = _rng(4)
    for _ in range(200):
        bb = r.choice([1, 2, 8])
        t = CacheTierParams(disk_bandwidth=r.choice([6e9, 2e9, 5e10]),
                            host_capacity_bytes=r.choice([64e9, 2e9, 5e8]),
                            window_batches=bb * r.randrange(1, 9), block_batches=bb)
        bpb = r.choice([1.2e8, 3.0e7, 1e6])
        if t.host_capacity_bytes < bb * bpb:
            continue
        n = r.randrange(1, 200)
        it = r.choice([0.0074, 0.045, 1e-4])
        assert prod.cache_tier_epoch(t, bpb, n, it) == ref.cache_tier_epoch(t, bpb, n, it)


def test_model_profiles(prod, ref):
    """Explicit specs built from geometry equal the reference presets."""
    vit = configs.model_spec(configs.GEOMETRIES["vit-b16"])
    preset = ref.model_preset("vit-b16")
    assert vit["attention_params"] == preset.attention_params
    assert vit["mlp_params"] == preset.mlp_params
    assert vit["activation_bytes"] == preset.activation_bytes
    assert preset.total_params() == 86_566_120
    big = ref.model_preset("bert-large")
    assert big.total_params() == 335_143_938
    g = configs.Geometry("bert", 24, 1024, 4096, 16, 512, 2)
    spec = configs.model_spec(g)
    assert spec["attention_params"] == big.attention_params
    assert spec["mlp_params"] == big.mlp_params
    assert spec["activation_bytes"] == big.activation_bytes
