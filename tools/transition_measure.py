"""Measured plan-transition overheads with two ranks
time-sharing one B200 (gloo, host-staged transfers): the planner's elastic
ViT-B/16 schedule compresses K = 2 -> 1 and forks a replica, and every epoch's
transition (parameter / momentum migration, DP regroup, AutoCache store
hand-over) is timed with CUDA events by Trainer.run_epoch.  Both ranks share
one GPU and move tensors through host memory, so the numbers are an upper
bound on what NVLink ranks would see; they sit beside the reference's Table-3
constants (runner.cpp:24-28).

    python tools/transition_measure.py [out.json]
"""
import json
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _scenario():
    from paper_2102_03161_b200 import configs
    s = configs.scenario("vit-b16", 2)
    s["training"]["per_pipeline_batch"] = 64
    s["training"]["epochs"] = 5
    s["training"]["alpha"] = 0.5
    s["cache"]["policy"] = "always_on"
    return s


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2102_03161_b200 import configs
        from paper_2102_03161_b200.trainer import Trainer
        torch.cuda.set_device(0)
        scen = _scenario()
        tr = Trainer(scen, configs.GEOMETRIES["vit-b16"], iterations_per_epoch=2, rank=rank,
                     world=world, device="cuda:0", host_staged=True, device_norms=False)
        rows = tr.run()
        if rank == 0:
            with open(out, "w") as f:
                json.dump([r.__dict__ for r in rows], f)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out",
                                                              "transitions.json")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    raw = out + ".rows"
    mp.spawn(_worker, args=(2, port, raw), nprocs=2, join=True)
    from paper_2102_03161_b200 import report
    from paper_2102_03161_b200.trainer import EpochResult
    rows = [EpochResult(**r) for r in json.load(open(raw))]
    table = report.transition_table(_scenario(), rows)
    res = {"setup": "2 ranks time-sharing one B200, gloo host-staged (upper bound)",
           "epochs": [{"epoch": r.epoch, "l_frozen": r.l_frozen, "k": r.k, "r": r.r,
                       "cache": r.cache_enabled, "transition_s": r.transition_time_s,
                       "iteration_s": r.iteration_time_s} for r in rows],
           "transitions": table}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))
