"""The real epoch loop (trainer.py) on the B200.

* With the scenario's synthetic norm source, the executed run takes exactly
  the reference's golden decisions (tests/golden, produced by the reference).
* With device norms, every freeze decision equals what the reference
  algorithm (oracle restatement, pinned in test_oracle_golden.py) decides for
  the norm vectors the device reported -- the trace-replay parity of
  SURVEY.md section 7.
* Two ranks (two processes sharing cuda:0, gloo) run an elastic schedule with
  a pipeline -> replica fork and agree on every decision.
"""
import json
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import eps_oracle as O
from paper_2102_03161_b200 import configs
from paper_2102_03161_b200.trainer import Trainer

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests/golden/decisions.json")))


def _tiny_scenario(gpus=1, batch=16, epochs=6, **kw):
    s = configs.scenario("tiny-vit", gpus)
    s["training"]["per_pipeline_batch"] = batch
    s["training"]["epochs"] = epochs
    s.update(kw)
    return s


def test_trainer_follows_golden_decisions(cuda):
    case = next(c for c in GOLDEN["scenarios"] if c["name"] == "tiny-vit-g1")
    scen = json.loads(json.dumps(case["scenario"]))
    scen["training"]["per_pipeline_batch"] = 16
    # the decisions do not depend on the batch here (K = R = M = 1 on one GPU)
    tr = Trainer(scen, configs.GEOMETRIES["tiny-vit"], iterations_per_epoch=2,
                 device_norms=False)
    rows = tr.run(6)
    for r, want in zip(rows, case["rows"]):
        assert (r.l_frozen, r.k, r.r, r.m, int(r.cache_enabled)) == (
            want["l_frozen"], want["pipeline_length"], want["replica_width"],
            want["micro_batches"], want["cache_enabled"])
        assert math_finite(r.mean_loss)
    assert Trainer.report_csv(rows).splitlines()[0].startswith("epoch,l_frozen,k,r,m,")


def math_finite(x):
    return x == x and abs(x) < 1e6


def test_device_norm_decisions_replay(cuda):
    scen = _tiny_scenario(epochs=5)
    g = configs.GEOMETRIES["tiny-vit"]
    tr = Trainer(scen, g, iterations_per_epoch=2, device_norms=True, lr=0.05)
    rows = tr.run()
    st = O.FreezeState(scen["training"]["alpha"])
    for e in range(1, len(rows)):
        norms = rows[e - 1].norms
        assert len(norms) == g.layers and all(n >= 0 for n in norms)
        assert O.next_frozen_count(st, norms, g.layers) == rows[e].l_frozen


def _elastic_scenario():
    # alpha 0.5 + cache always on: K=2 pipeline, cache write 0->2 under K=2,
    # then compression to K=1 with a forked replica (R=2), cache move 2->3,
    # then steady cache gathers -- every transition of the run loop
    s = _tiny_scenario(gpus=2, batch=8, epochs=5)
    s["training"]["alpha"] = 0.5
    s["cache"]["policy"] = "always_on"
    return s


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, tier="hbm", peer=False, autodp=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scen = _elastic_scenario()
        scen["features"]["autodp"] = autodp
        tr = Trainer(scen, configs.GEOMETRIES["tiny-vit"], iterations_per_epoch=3, rank=rank,
                     world=world, device="cuda:0", host_staged=True, device_norms=False,
                     cache_tier=tier, peer=peer)
        rows = []
        for e in range(5):
            rows.append(tr.run_epoch(e))
            if e == 1:
                store_bytes = tr.store.shard_bytes()
        tr.close()
        torch.save({"rows": [(r.l_frozen, r.k, r.r, r.m, r.cache_enabled, r.mean_loss,
                              r.samples) for r in rows],
                    "csv": Trainer.report_csv(rows), "store_bytes": store_bytes,
                    "dataset": tr.dataset},
                   os.path.join(out, f"tr_{rank}.pt"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tier,peer,autodp", [("hbm", False, True), ("host", False, True),
                                              ("hbm", True, True), ("hbm", False, False),
                                              ("disk", False, True)])
def test_two_rank_elastic_run(cuda, tmp_path, tier, peer, autodp):
    """Two ranks run the elastic schedule: K 2 -> 1 with a replica fork (or,
    AutoDP off, with the freed GPU idle -- runner.cpp:445), cache writes into
    the node-sharded store (HBM: each rank holds half the rows, peers'
    rows over IPC) or the shared host segment, measured CSV columns."""
    mp.spawn(_worker, args=(2, _port(), str(tmp_path), tier, peer, autodp), nprocs=2, join=True)
    ra, rb = (torch.load(tmp_path / f"tr_{r}.pt") for r in range(2))
    a, b = ra["rows"], rb["rows"]
    assert [x[:5] for x in a] == [x[:5] for x in b]
    ks = [x[1] for x in a]
    assert ks == [2, 2, 1, 1, 1]
    assert [x[2] for x in a] == ([1, 1, 2, 2, 2] if autodp else [1, 1, 1, 1, 1])
    assert [x[4] for x in a] == [False, True, True, True, True]
    assert all(x[6] == ra["dataset"] for x in a)  # every sample trained every epoch
    # the planner packs 2 stages into 1 and forks a second replica at some epoch
    from paper_2102_03161_b200 import LIB_PATH
    from paper_2102_03161_b200.capi import EpsApi
    from paper_2102_03161_b200.planner import Planner
    sc = _elastic_scenario()
    sc["features"]["autodp"] = autodp
    pl = Planner(EpsApi(LIB_PATH, "eps_"), sc)
    want = [pl.begin_epoch(e) for e in range(5)]
    assert ks == [d.pipeline_length for d in want]
    assert [x[0] for x in a] == [d.l_frozen for d in want]
    for x in a + b:
        if x[5] == x[5]:  # last-stage ranks report a loss
            assert 0 < x[5] < 20
    g = configs.GEOMETRIES["tiny-vit"]
    row = g.tokens * g.hidden * 2
    if tier == "hbm":  # per-GPU store bytes ~ dataset / world
        assert ra["store_bytes"] == rb["store_bytes"] == -(-ra["dataset"] // 2) * row
    else:  # one node-wide segment / file
        assert ra["store_bytes"] == ra["dataset"] * row
    lines = ra["csv"].splitlines()
    assert len(lines) == 6 and all(len(ln.split(",")) == 15 for ln in lines)


def _shard_worker(rank, world, port, out):
    """Each rank scatters the rows it 'processed' into the node-sharded store
    (half of them land on the peer's HBM over IPC), then gathers every row."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ctypes as C
        from paper_2102_03161_b200 import ops
        from paper_2102_03161_b200.trainer import CacheStore
        torch.cuda.set_device(0)
        n, elems = 13, 96
        st = CacheStore("hbm", n, elems, rank, world, torch.device("cuda:0"), collective=True)
        mine = torch.arange(rank, n, world, device="cuda:0")
        src = (mine.to(torch.float32)[:, None] * 1000 +
               torch.arange(elems, device="cuda:0")[None, :]).to(torch.bfloat16)
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ops.call("eps_cache_scatter_sharded", st.table, C.c_int64(st.rows_per_shard), mine,
                 mine.numel(), C.c_int64(elems * 2), src, s)
        torch.cuda.synchronize()
        dist.barrier()
        got = st.rows(torch.arange(n, device="cuda:0"))
        torch.cuda.synchronize()
        torch.save({"got": got.cpu(), "local_rows": st.local.shape[0]},
                   os.path.join(out, f"sh_{rank}.pt"))
        dist.barrier()
        st.close()
    finally:
        dist.destroy_process_group()


def test_sharded_store_peer_gather(cuda, tmp_path):
    mp.spawn(_shard_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    want = (torch.arange(13, dtype=torch.float32)[:, None] * 1000 +
            torch.arange(96)[None, :]).to(torch.bfloat16)
    for r in range(2):
        o = torch.load(tmp_path / f"sh_{r}.pt")
        assert o["local_rows"] == 7  # ceil(13 / 2) rows per GPU
        assert torch.equal(o["got"], want)


def test_measured_timeline_blocks(cuda):
    """StageRunner.trace: the last iteration's F / B blocks in the reference's
    timeline schema (runner.cpp:357-367), ordered and non-overlapping."""
    scen = _tiny_scenario(epochs=1)
    tr = Trainer(scen, configs.GEOMETRIES["tiny-vit"], iterations_per_epoch=2)
    tr.runner.trace = []
    tr.run(1)
    tl = tr.runner.timeline()
    assert [b["kind"] for b in tl] == ["F", "B"]
    assert set(tl[0]) == {"device", "kind", "start_s", "end_s", "tag"}
    assert 0.0 <= tl[0]["start_s"] < tl[0]["end_s"] <= tl[1]["start_s"] < tl[1]["end_s"]


def test_host_tier_prefetch_window_matches_hbm_tier(cuda):
    """the host tier's gather epochs read their cached
    boundary activations through the prefetch window (copy-stream gathers into
    HBM staging, one iteration ahead).  Same bytes reach the executor, so every
    epoch's loss and gradient norms equal the HBM tier's and the unwindowed
    host tier's exactly."""
    scen = _tiny_scenario(epochs=5)
    scen["training"]["alpha"] = 0.5
    scen["cache"]["policy"] = "always_on"
    g = configs.GEOMETRIES["tiny-vit"]
    # the window stages exactly the store's rows (bitwise)
    tr = Trainer(scen, g, iterations_per_epoch=3, device_norms=False, cache_tier="host",
                 cache_prefetch=True)
    rows = [tr.run_epoch(e) for e in range(5)]
    last = rows[-1]
    assert last.cache_enabled and not last.cache_moved
    _, shards = tr.api.redistribute(tr.dataset, tr.cluster, last.k, last.epoch, tr.seed)
    ids = torch.tensor(shards[0], dtype=torch.int64, device="cuda")
    n_its = len(shards[0]) // tr.batch
    ids_last = ids[(n_its - 1) * tr.batch:n_its * tr.batch]
    torch.cuda.synchronize()
    assert torch.equal(tr._win_buf[(n_its - 1) % 2], tr.store.rows(ids_last))
    tr.close()
    runs = {}
    for name, kw in {"hbm": dict(cache_tier="hbm"),
                     "host": dict(cache_tier="host", cache_prefetch=False),
                     "host+window": dict(cache_tier="host", cache_prefetch=True)}.items():
        tr = Trainer(scen, g, iterations_per_epoch=3, device_norms=False, **kw)
        runs[name] = [(r.l_frozen, r.cache_enabled, r.cache_moved, r.mean_loss, tuple(r.norms))
                      for r in tr.run()]
    assert any(r[1] and not r[2] for r in runs["hbm"])  # some epochs are pure gathers
    for name in ("host", "host+window"):
        for a, b in zip(runs[name], runs["hbm"]):
            assert a[:3] == b[:3]
            # bias-gradient reductions use float atomics (run-to-run order), so
            # equal inputs agree to rounding, not bit for bit (the staged rows
            # themselves are checked bitwise above)
            assert abs(a[3] - b[3]) <= 1e-3 * abs(b[3])
            assert all(abs(x - y) <= 1e-2 * max(abs(y), 1e-6) for x, y in zip(a[4], b[4]))


def test_disk_tier_matches_hbm_tier(cuda, tmp_path):
    """SURVEY.md 8(f) row 1, the disk level: the cached boundary activations
    live in a file behind the DiskTier host window (CacheTierSim's disk ->
    host prefetch, autocache.cpp:69-150, executed).  The staged rows equal the
    file's rows bitwise, and every epoch's decisions, loss and norms equal the
    HBM tier's (to the float-atomic rounding of the bias gradients)."""
    scen = _tiny_scenario(epochs=5)
    scen["training"]["alpha"] = 0.5
    scen["cache"]["policy"] = "always_on"
    scen["cache"]["window_batches"] = 2  # a sliding window: 3 batches per epoch
    scen["cache"]["block_batches"] = 1
    g = configs.GEOMETRIES["tiny-vit"]
    tr = Trainer(scen, g, iterations_per_epoch=3, device_norms=False, cache_tier="disk",
                 cache_dir=str(tmp_path))
    rows = [tr.run_epoch(e) for e in range(5)]
    last = rows[-1]
    assert last.cache_enabled and not last.cache_moved
    _, shards = tr.api.redistribute(tr.dataset, tr.cluster, last.k, last.epoch, tr.seed)
    ids = torch.tensor(shards[0], dtype=torch.int64, device="cuda")
    n_its = len(shards[0]) // tr.batch
    ids_last = ids[(n_its - 1) * tr.batch:n_its * tr.batch]
    torch.cuda.synchronize()
    staged = tr._win_buf[(n_its - 1) % 2].clone()
    assert torch.equal(staged, tr.store.rows(ids_last))
    st = [s for s in tr.disk_stats if s["mode"] == 1]
    assert st and st[-1]["bytes_read"] > 0 and st[-1]["evictions"] >= 3
    assert st[-1]["max_resident_bytes"] <= 2 * tr.batch * tr.store.disk.stride
    assert any(s["bytes_written"] > 0 for s in tr.disk_stats)
    path = tr.store.path
    tr.close()
    assert not os.path.exists(path)
    hbm = Trainer(scen, g, iterations_per_epoch=3, device_norms=False, cache_tier="hbm")
    ref = hbm.run()
    for a, b in zip(rows, ref):
        assert (a.l_frozen, a.cache_enabled, a.cache_moved) == (b.l_frozen, b.cache_enabled,
                                                                b.cache_moved)
        assert abs(a.mean_loss - b.mean_loss) <= 1e-3 * abs(b.mean_loss)
        assert all(abs(x - y) <= 1e-2 * max(abs(y), 1e-6) for x, y in zip(a.norms, b.norms))
