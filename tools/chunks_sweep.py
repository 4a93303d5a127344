"""The chunks (micro-batch count) sweep of cli.cpp:96-117 measured on one
B200: ViT-B/16, batch 400, K = 1, M = 1..6 -- the
executed iteration (fwd + bwd + SGD over M sequential micro-batches) beside
the reference's modeled times, raw and with the B200-calibrated c_fwd.

    python tools/chunks_sweep.py [out.json] [iters]
"""
import dataclasses
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2102_03161_b200 import LIB_PATH, configs, report  # noqa: E402
from paper_2102_03161_b200.capi import EpsApi  # noqa: E402
from paper_2102_03161_b200.trainer import Trainer  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/chunks_sweep.json"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
api = EpsApi(LIB_PATH, "eps_")
scen = configs.scenario("vit-b16", 1)
geom = configs.GEOMETRIES["vit-b16"]
tr = Trainer(scen, geom, iterations_per_epoch=2, device_norms=False)
tr.run_epoch(0)  # epoch-0 plan (L_f = 0, K = 1), kernels configured
base = tr.runner.plan
ids = torch.arange(tr.batch, device=tr.device)
x, y = tr.images.index_select(0, ids), tr.labels.index_select(0, ids)


def run_m(m):
    tr.runner.set_plan(dataclasses.replace(base, M=m))

    def one():
        tr.runner.iteration(x, y, tr.batch)
        tr.runner.sync_grads()
        tr.runner.step(tr.lr, tr.momentum)

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        one()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters / 1000.0


t1 = run_m(1)
cal = report.calibrate_c_fwd(api, scen, t1)
rows = report.chunks_sweep(api, scen, 1, run_m, calibrated_c_fwd=cal["c_fwd"])
# the interconnect sweep (cli.cpp:118-127) of the 2 x 8 scenario, replayed with
# the B200 forward rate measured above (one GPU cannot vary its interconnect)
two_nodes = configs.scenario("vit-b16", 8)
two_nodes["cluster"]["nodes"] = 2  # 2 nodes x 8 GPUs: the replicas' all-reduce crosses nodes
bw = report.bandwidth_sweep(api, two_nodes, [1e9, 5e9, 12.5e9, 25e9, 50e9, 100e9],
                            calibrated_c_fwd=cal["c_fwd"])
with open(out, "w") as f:
    json.dump({"device": torch.cuda.get_device_name(), "iters": iters,
               "calibrated_c_fwd": cal["c_fwd"], "rows": rows, "bandwidth_sweep_2x8": bw}, f,
              indent=1)
for r in rows:
    print(json.dumps(r))
