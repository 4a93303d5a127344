"""SURVEY.md 8(f) rows 3-4 on a multi-GPU node: the measured feature ladder
(runner.cpp:307-338: baseline / freeze / autopipe / autopipe+autocache /
autopipe+autodp / all), the micro-batch-count (chunks) sweep at K = N, and
the plan-transition overheads of the elastic schedule (Table 3,
runner.cpp:22-28, charged at runner.cpp:157) -- each rung executed by
`Trainer` (device gradient norms -> reference planner -> NCCL communicator
plane, peer-memory stage hand-off) with the modeled numbers beside it.

    torchrun --nnodes 1 --nproc-per-node N --master-addr 127.0.0.1 \
        tools/multi_gpu_sweeps.py [cfg] [iters_per_epoch] [epochs] [out.json]

One process per GPU (RANK / LOCAL_RANK / WORLD_SIZE from torchrun); rank 0
writes the JSON.  Runs at N = 1 as well (the CI check of this harness on the
one-GPU sandbox); the multi-GPU numbers need a multi-GPU box.
"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2102_03161_b200 import LIB_PATH, configs, report  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.trainer import Trainer  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "vit-b16"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    epochs = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    out_path = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out",
                                                                  "multi_gpu_sweeps.json")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    g = configs.GEOMETRIES[cfg]
    base = configs.scenario(cfg, world)
    base["training"]["epochs"] = epochs
    api = EpsApi(LIB_PATH, "eps_")
    comm = "eps" if world > 1 else "torch"
    peer = world > 1

    def run(scen):
        tr = Trainer(scen, g, iterations_per_epoch=iters, rank=rank, world=world, device=dev,
                     comm=comm, peer=peer)
        rows = tr.run()
        del tr
        torch.cuda.empty_cache()
        return rows

    out = {"cfg": cfg, "world": world, "iterations_per_epoch": iters, "epochs": epochs,
           "comm": comm, "peer_handoff": peer, "gpu": torch.cuda.get_device_name(dev)}
    t0 = time.time()
    # feature ladder (measured total incl. transitions vs the modeled ladder)
    totals = {}

    def rung_total(scen):
        rows = run(scen)
        t = sum(r.epoch_time_s + r.transition_time_s for r in rows)
        totals[json.dumps(scen["features"], sort_keys=True)] = rows
        return t

    out["ladder"] = report.ladder(api, base, rung_total, rungs=[n for n, _ in report.LADDER])
    # transition overheads of the full run (every epoch's set_plan, measured)
    full = totals[json.dumps(report.with_features(base, dict(report.LADDER)["all"])["features"],
                             sort_keys=True)]
    out["transitions"] = [{"epoch": r.epoch, "K": r.k, "R": r.r, "l_frozen": r.l_frozen,
                           "cache_moved": r.cache_moved, "transition_s": r.transition_time_s,
                           "cache_transition_s": r.cache_transition_time_s,
                           "comm_s": r.comm_time_s, "exposed_comm_s": r.exposed_comm_time_s,
                           "bubble_s": r.bubble_time_s, "stall_s": r.stall_time_s}
                          for r in full]
    out["reference_transition_constants"] = base["cost_model"].get("transition_overheads", {})
    # chunks sweep at the epoch-0 pipeline length (K = N, cli.cpp:96-117): the
    # executed iteration for every M in [K, 6K] beside optimal_chunks' model
    import dataclasses
    tr = Trainer(base, g, iterations_per_epoch=2, rank=rank, world=world, device=dev,
                 comm=comm, peer=peer, device_norms=False)
    tr.run_epoch(0)
    plan0 = tr.runner.plan
    ids = torch.arange(tr.batch, device=dev)
    x, y = tr.images.index_select(0, ids), tr.labels.index_select(0, ids)

    def run_m(m):
        tr.runner.set_plan(dataclasses.replace(plan0, M=m))

        def one():
            tr.runner.iteration(x if tr.runner.stage == 0 else None, y, tr.batch)
            tr.runner.sync_grads()
            tr.runner.step(tr.lr, tr.momentum)

        for _ in range(2):
            one()
        tr._barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            one()
        b.record()
        tr._barrier()
        return tr._max_over_ranks(a.elapsed_time(b) / 4 / 1e3)

    out["chunks_sweep"] = report.chunks_sweep(api, base, plan0.K, run_m)
    tr.close()
    out["wall_s"] = time.time() - t0
    if rank == 0:
        os.makedirs(os.path.dirname(out_path), exist_ok=True)
        with open(out_path, "w") as f:
            json.dump(out, f, indent=1)
        print(json.dumps({k: v for k, v in out.items() if k != "transitions"})[:2000])
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
