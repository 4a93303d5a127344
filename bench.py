"""Benchmark: ViT-B/16 freeze-training samples/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one training iteration of the per-pipeline batch (400 synthetic
224x224 ImageNet-shaped images, BASELINE.json configs[1]): forward, backward
and the fused SGD-momentum update of every trainable layer, executed by the
sm_100a kernels of libeps_b200.so through the C ABI.  The epoch-0 decision
of the reference's planner (runner.cpp:94-229, replayed by eps_planner) fixes
L_frozen = 0, K, R and M; `value` is that no-freeze step's whole-job
throughput with inputs resident in HBM.  `e2e` is the same step through the
public executor API with the images copied from pinned host memory every
step and the loss read back.  `freeze_schedule` replays the planner's
per-epoch decisions (L_frozen, AutoCache gather / boundary move) on the
device and reports the measured end-to-end speedup vs no-freeze
(runner.cpp:298 semantics: baseline total time / freeze total time).

N > 1 (torchrun, one rank per GPU, NCCL): the ranks execute the planner's
plan -- K-stage GPipe pipelines times R AutoDP replicas (per-stage NCCL
all-reduce of the active gradients in 25 MB buckets during the drain).  The
stage hand-off (--p2p ipc, default) is fused into the producing kernels: the
last GEMM / LayerNorm of a stage stores the cut activation straight into the
next stage's buffer over CUDA-IPC peer memory (NVLink), and the gradient
flows back the same way, ordered by stream flags; --p2p nccl uses NCCL
send / recv instead.  At epoch 0 the reference plans K = N, R = 1, so
the per-step work is one 400-image batch at every N ("scaling": "strong");
the freeze schedule forks replicas as layers freeze.

`--impl reference` times the reference path's CPU implementation -- the fp32
restatement in oracle/vit_fp32.py (the reference itself has no tensor code,
SURVEY.md section 0) -- on the host cores, on a bounded sample of the same
workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

CFG = "vit-b16"
METRIC = "ViT-B/16 train samples/sec"
UNIT = "samples/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CFG)
    ap.add_argument("--no-schedule", action="store_true", help="skip the freeze-schedule replay")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--p2p", default="ipc", choices=["ipc", "nccl"],
                    help="stage hand-off: producer kernels write the neighbour's buffers over "
                         "CUDA-IPC peer memory (default) or NCCL send/recv")
    ap.add_argument("--gloo-one-gpu", action="store_true",
                    help="test mode: all ranks share cuda:0, gloo with host-staged transfers")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---- clocks sampling (B200_PROFILING.md clocks line) -------------------------
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


def layer_flops(g) -> float:
    """F = 2T(4d^2 + 2df) + 4T^2 d per sample per layer (forward)."""
    T, d, f = g.tokens, g.hidden, g.mlp_dim
    return 2.0 * T * (4 * d * d + 2 * d * f) + 4.0 * T * T * d


def sample_flops(g, l_frozen: int = 0, cached: bool = False) -> float:
    """Algorithmic training FLOPs per sample; embedding / head
    counted as their GEMMs (3x trainable, 1x frozen)."""
    F = layer_flops(g)
    L = g.layers
    n_patch = (g.image // g.patch) ** 2
    embed = 2.0 * n_patch * g.hidden * g.channels * g.patch * g.patch
    head = 2.0 * g.hidden * g.classes
    total = 3.0 * head
    for l in range(L):
        if l >= l_frozen:
            total += (2.0 if (l == l_frozen and l_frozen > 0) else 3.0) * F
        elif not cached:
            total += F
    if l_frozen == 0:
        total += 3.0 * embed
    elif not cached:
        total += embed
    return total


# ---- reference arm -------------------------------------------------------------
def cpu_baseline(g, seconds: float, batch: int = 4):
    """fp32 CPU restatement of the train step (oracle/vit_fp32.py) on the host
    cores: samples/sec over a bounded sample of `batch`-image steps."""
    from oracle import vit_fp32
    from paper_2102_03161_b200.vit import init_params
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    params = init_params(g, seed=17)
    gen = torch.Generator().manual_seed(5)
    images = torch.randn(batch, g.channels, g.input_image, g.input_image, generator=gen)
    labels = torch.randint(0, g.classes, (batch,), generator=gen)
    vit_fp32.train_step(params, images, labels, g, 0)  # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        _, grads, _ = vit_fp32.train_step(params, images, labels, g, 0)
        with torch.no_grad():
            for k in params:
                params[k] -= 1e-3 * grads[k]
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return {"value": n * batch / el, "unit": UNIT, "cores": torch.get_num_threads(),
            "kind": "port",
            "sample": f"{n} steps x {batch} images of the {g.image}px ViT-B/16 train step "
                      f"(fp32, forward+backward+SGD) in {el:.1f}s"}


def run_reference(args, world, rank):
    from paper_2102_03161_b200.configs import GEOMETRIES, BATCH
    if rank != 0:
        return
    g = GEOMETRIES[args.config]
    # warm-up + K steps of the bounded sample, timed as one window
    cb = cpu_baseline(g, args.cpu_seconds)
    v = cb["value"]
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * BATCH[args.config] / v,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic",
           "config": {"workload": f"{args.config} 224px batch {BATCH[args.config]} train step "
                                  "(bounded CPU sample)", "global_batch": BATCH[args.config] *
                      max(1, args.gpus), "seq_len": g.tokens, "parallelism": "cpu"},
           "cpu_baseline": cb,
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---- our arm -------------------------------------------------------------------
def main_ours(args, world, rank, local):
    from paper_2102_03161_b200 import LIB_PATH, configs, ops
    from paper_2102_03161_b200.capi import EpsApi
    from paper_2102_03161_b200.pipeline import StagePlan, StageRunner, Transport
    from paper_2102_03161_b200.planner import Planner
    from paper_2102_03161_b200.vit import VitExecutor

    one_gpu = args.gloo_one_gpu
    dev = torch.device("cuda", 0 if one_gpu else local)
    torch.cuda.set_device(dev)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    g = configs.GEOMETRIES[args.config]
    batch = configs.BATCH[args.config]
    scen = configs.scenario(args.config, world)
    planner = Planner(EpsApi(LIB_PATH, "eps_"), scen)
    decisions = [planner.begin_epoch(e) for e in range(configs.EPOCHS[args.config])]
    plan0 = StagePlan.from_decision(decisions[0], g.layers)

    ex = VitExecutor(g, max_batch=batch, seed=17, device=dev)
    runner = StageRunner(ex, rank, world, Transport(host_staged=one_gpu),
                         peer=(args.p2p == "ipc"))
    runner.set_plan(plan0)
    pipe, stage = plan0.role(rank)
    gen = torch.Generator(device=dev).manual_seed(1234 + pipe)
    images = torch.randn(batch, g.channels, g.input_image, g.input_image, device=dev,
                         generator=gen)
    labels = torch.randint(0, g.classes, (batch,), device=dev, generator=gen)
    stream = torch.cuda.current_stream()

    def step(imgs, cache_mode=0, cache_old=0, store=None, ids=None, lbls=None):
        loss = runner.iteration(imgs, labels if lbls is None else lbls, batch,
                                cache_mode=cache_mode, cache_old=cache_old, store=store, ids=ids)
        runner.sync_grads()
        runner.step(lr=1e-3, momentum=0.9)
        return loss

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(x: float, op) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if one_gpu else dev, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def timed(fn, steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        s.record(stream)
        for _ in range(steps):
            fn()
        e.record(stream)
        barrier()
        return reduce(s.elapsed_time(e), dist.ReduceOp.MAX if world > 1 else None) / steps

    # ---- value: the epoch-0 (no-freeze) iteration, inputs resident in HBM ------
    for _ in range(args.warmup):
        step(images)
    clocks = ClockSampler(dev.index)
    clocks.start()
    n_launch0 = ops.launch_count()
    ms = timed(lambda: step(images), args.steps)
    launches = int(reduce(float(ops.launch_count() - n_launch0),
                          dist.ReduceOp.SUM if world > 1 else None))
    clock_rec = clocks.stop()
    value = plan0.R * batch / (ms / 1000.0)

    # ---- roofline: instrumented steps, per-class CUDA-event times --------------
    # three instrumented steps; per class the median device time (one step is
    # exposed to a single power-cap excursion)
    reps = []
    for _ in range(3):
        ex.timing(True)
        step(images)
        torch.cuda.synchronize()
        reps.append(ex.timing_read())
        ex.timing(False)
    cls = {name: dict(reps[0][name], ms=sorted(r[name]["ms"] for r in reps)[1])
           for name in reps[0]}
    for c in cls.values():  # whole-job sums (every rank's launches)
        for k in ("ms", "flops", "bytes", "launches"):
            c[k] = reduce(float(c[k]), dist.ReduceOp.SUM if world > 1 else None)
    peaks, peak_kind = measured_peaks()
    gemm = cls["gemm"]
    gemm_tflops = gemm["flops"] / (gemm["ms"] / 1000.0) / 1e12
    peak_tc = peaks["bf16_tflops_sustained"]
    roofline = {"bound": "tensor", "kernel": "eps_k::gemm_tc_kernel (all block GEMMs of a step)",
                "achieved": round(gemm_tflops, 1), "peak": peak_tc, "unit": "TFLOP/s",
                "frac": round(gemm_tflops / peak_tc, 4), "traffic": None,
                "peak_kind": f"{peak_kind} bf16_tflops_sustained",
                "launches_per_step": int(gemm["launches"]),
                "share_of_step": round(gemm["ms"] / sum(c["ms"] for c in cls.values()), 4)}
    # DRAM traffic per GEMM launch from the committed ncu --set full capture
    # (tools/gemm_traffic.py; layer-1 forward QKV / proj / FC1 / FC2 launches)
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            tr = json.load(f)
        roofline["traffic"] = round(tr["mean_dram_bytes_per_launch"])
        roofline["traffic_note"] = ("dram bytes per launch, mean of the profiled launches in "
                                    "profiles/gemm_traffic.json")
    except (OSError, KeyError, ValueError):
        pass
    kernels = {}
    for name, c in cls.items():
        if c["launches"] == 0:
            continue
        k = {"ms_per_step": round(c["ms"] / world, 3), "launches": int(c["launches"])}
        if c["flops"]:
            k["tflops"] = round(c["flops"] / (c["ms"] / 1000.0) / 1e12, 1)
        if c["bytes"]:
            k["gbs"] = round(c["bytes"] / (c["ms"] / 1000.0) / 1e9, 1)
            k["hbm_frac"] = round(k["gbs"] / peaks["hbm_gbs"], 4)
        kernels[name] = k
    mfu = sample_flops(g) * value / world / 1e12 / peak_tc

    # ---- e2e: host-pinned inputs copied every step, loss read back -------------
    # A training loop's input pipeline: step i+1's batch is copied H2D on a copy
    # stream (double-buffered) while step i computes, and step i's loss is read
    # back through a pinned buffer one step later, so the host never stalls the
    # device.  Every step still moves its own inputs and result across PCIe.
    h_images = images.cpu().pin_memory()
    h_labels = labels.cpu().pin_memory()
    first, last = stage == 0, stage == plan0.K - 1
    h2d = (h_images.numel() * 4 + h_labels.numel() * 8) * plan0.R
    d_img = [torch.empty_like(images) for _ in range(2)]
    d_lab = [torch.empty_like(labels) for _ in range(2)]
    h_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()
    h2d_done, used, d2h_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
    state = {"i": 0, "losses": []}

    def prefetch(slot):
        copy_stream.wait_event(used[slot])
        with torch.cuda.stream(copy_stream):
            if first:
                d_img[slot].copy_(h_images, non_blocking=True)
            if last:
                d_lab[slot].copy_(h_labels, non_blocking=True)
            h2d_done[slot].record(copy_stream)

    prefetch(0)

    def e2e_step():
        i = state["i"]
        slot = i % 2
        stream.wait_event(h2d_done[slot])
        loss = step(d_img[slot], lbls=d_lab[slot])
        used[slot].record(stream)
        if last:
            h_loss[slot].copy_(loss, non_blocking=True)
        d2h_done[slot].record(stream)
        prefetch(1 - slot)
        if i > 0:  # previous step's loss, read while this one runs
            d2h_done[1 - slot].synchronize()
            state["losses"].append(float(h_loss[1 - slot].item()))
        state["i"] = i + 1

    for _ in range(2):
        e2e_step()
    e2e_ms = timed(e2e_step, args.steps)
    e2e_value = plan0.R * batch / (e2e_ms / 1000.0)

    # ---- freeze schedule: the planner's per-epoch decisions on the device ------
    sched = None
    if not args.no_schedule:
        sched = freeze_schedule(runner, g, batch, decisions, images, step, timed, ms, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(g, args.cpu_seconds)

    if rank == 0:
        par = f"pipe{plan0.K}" + (f"xdp{plan0.R}" if plan0.R > 1 else "")
        out = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
               "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
               "vs_baseline": None,
               "dtype": "bf16", "data": "synthetic (seeded N(0,1) images, U[0,1000) labels; "
                                         "random trunc-normal weights)",
               "config": {"workload": f"{args.config}: ViT-B/16 224px, batch {batch} per "
                                      "pipeline, no-freeze iteration (fwd+bwd+SGD) under the "
                                      "reference planner's epoch-0 plan",
                          "model": "ViT-B/16", "global_batch": batch * plan0.R,
                          "seq_len": g.tokens, "parallelism": par,
                          "planner": {"K": plan0.K, "R": plan0.R, "M": plan0.M,
                                      "spans": [list(x) for x in plan0.spans]},
                          "l2": "working set (>20 GB of activations) far exceeds the 126 MB L2"},
               "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": 4 * plan0.R, "ms_per_step": round(e2e_ms, 3)},
               "gpu_launches": launches,
               "roofline": roofline,
               "kernels": kernels,
               "mfu": round(mfu, 4),
               "clocks": clock_rec,
               "freeze_schedule": sched,
               "cpu_baseline": cpu}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def freeze_schedule(runner, g, batch, decisions, images, step, timed, ms0, dev):
    """Per-epoch steady-state iteration time under the planner's decisions.

    Epoch e runs L_frozen(e) on its K(e)-stage pipelines x R(e) replicas (the
    runner migrates weights and regroups on every plan change) with the
    frozen prefix either recomputed (cache off), gathered from the HBM store
    (cache on) or -- on a boundary-move epoch -- gathered from the old
    boundary, forwarded over [old, new) and scattered at the new one
    (autocache.cpp:45-67).  An epoch holds the same samples at every width,
    so its time is proportional to t_e / R_e; speedup vs no-freeze (K0, R0,
    all layers trained: runner.cpp:67-90, 298) = sum_e t_0/R_0 / sum_e t_e/R_e."""
    from paper_2102_03161_b200.pipeline import StagePlan
    store = torch.zeros(batch, g.tokens * g.hidden, dtype=torch.bfloat16, device=dev)
    ids = torch.randperm(batch, generator=torch.Generator().manual_seed(3)).to(dev)
    memo, rows = {}, []
    r0 = decisions[0].replica_width
    for d in decisions:
        plan = StagePlan.from_decision(d, g.layers)
        if not d.cache_enabled:
            mode, old = 0, 0
        elif d.cache_moved:
            mode, old = 2, d.cache_old_boundary
        else:
            mode, old = 1, 0
        key = (plan, mode, old)
        if key not in memo:
            runner.set_plan(plan)
            if mode == 1:  # fill the store at this boundary first
                step(images, 2, 0, store, ids)
            fn = lambda: step(images, mode, old, store if mode else None, ids if mode else None)
            fn()
            memo[key] = timed(fn, 3)
        t = memo[key]
        rows.append({"epoch": d.epoch, "l_frozen": d.l_frozen, "K": plan.K, "R": plan.R,
                     "M": plan.M, "cache": ["off", "move", "gather"][[0, 2, 1].index(mode)],
                     "ms_per_iteration": round(t, 3),
                     "samples_per_s": round(plan.R * batch / (t / 1000.0), 1)})
    base = sum(ms0 / r0 for _ in rows)
    tot = sum(r["ms_per_iteration"] / r["R"] for r in rows)
    return {"epochs": rows, "no_freeze_ms_per_iteration": round(ms0, 3),
            "speedup_vs_no_freeze": round(base / tot, 4),
            "note": "per-epoch decisions from the reference planner, each executed on the "
                    "device (K-stage pipelines x R replicas)"}


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    main_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
