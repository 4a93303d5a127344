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
UNIT = "samples/s"

# BASELINE.json configs benchmarked by `--config` (the default is the metric's
# ViT-B/16 224 config; the others are configs[2..4] and the tiny config 0).
WORKLOADS = {
    "vit-b16": ("ViT-B/16 train samples/sec", "ViT-B/16 224px, batch 400 per pipeline"),
    "vit-b16-cifar100": ("ViT-B/16 CIFAR-100-shaped train samples/sec",
                         "ViT-B/16, 32px CIFAR-shaped input upsampled on device to 224, 100 "
                         "classes, batch 320 per pipeline"),
    "bert-base-384": ("BERT-base seq-384 SQuAD train samples/sec",
                      "BERT-base, 384 tokens, SQuAD span head, batch 64 per pipeline"),
    "bert-large-128": ("BERT-large seq-128 GLUE train samples/sec",
                       "BERT-large, 128 tokens, pooled 2-class head, batch 64 per pipeline"),
    "tiny-vit": ("tiny ViT train samples/sec",
                 "tiny ViT (4 x d128, p4, T65), 32px input, batch 64"),
}


def metric_of(cfg: str) -> str:
    return WORKLOADS[cfg][0]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CFG, choices=sorted(WORKLOADS))
    ap.add_argument("--no-schedule", action="store_true", help="skip the freeze-schedule replay")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-energy", action="store_true", help="skip the ~2 s energy run")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-trainer", action="store_true",
                    help="skip the real epoch-loop (Trainer) freeze vs no-freeze run")
    ap.add_argument("--trainer-iters", type=int, default=3,
                    help="iterations per epoch of the real epoch-loop run")
    ap.add_argument("--no-stage-emulation", action="store_true",
                    help="skip the single-GPU emulation of a K = 8 pipeline stage")
    ap.add_argument("--p2p", default="ipc", choices=["ipc", "nccl"],
                    help="stage hand-off: producer kernels write the neighbour's buffers over "
                         "CUDA-IPC peer memory (default) or NCCL send/recv")
    ap.add_argument("--comm", default="eps", choices=["eps", "torch"],
                    help="N > 1 collectives / sends: the library's NCCL communicator plane "
                         "(eps_comm_*, default) or torch.distributed's NCCL process groups")
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

    def energy_mj(self):
        # NVML total-energy counter (mJ since driver load); None when unavailable
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            return float(pynvml.nvmlDeviceGetTotalEnergyConsumption(h))
        except Exception:  # noqa: BLE001 -- optional telemetry
            return None

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
    counted as their GEMMs (3x trainable, 1x frozen; BERT's embedding is a
    gather, no GEMM)."""
    F = layer_flops(g)
    d = g.hidden
    if g.kind == "vit":
        embed = 2.0 * (g.image // g.patch) ** 2 * d * g.channels * g.patch * g.patch
        head = 2.0 * d * g.classes
    else:
        embed = 0.0
        head = (2.0 * g.tokens * d * g.classes if g.head == "qa"
                else 2.0 * d * g.classes + (2.0 * d * d if g.pooler else 0.0))
    total = 3.0 * head
    for l in range(g.layers):
        if l >= l_frozen:
            total += (2.0 if (l == l_frozen and l_frozen > 0) else 3.0) * F
        elif not cached:
            total += F
    if l_frozen == 0:
        total += 3.0 * embed
    elif not cached:
        total += embed
    return total


def synthetic_inputs(g, batch: int, gen, device):
    """(inputs, labels) of the synthetic workload: ViT images N(0,1) [B,3,S,S]
    + labels U[0,C); BERT token ids U[0,vocab) / segment ids (second half 1)
    as int64 [2,B,T] + labels (QA: start then end positions U[0,T), [2B])."""
    if g.kind == "vit":
        x = torch.randn(batch, g.channels, g.input_image, g.input_image, device=device,
                        generator=gen)
        y = torch.randint(0, g.classes, (batch,), device=device, generator=gen)
        return x, y
    tok = torch.randint(0, g.vocab, (batch, g.tokens), device=device, generator=gen)
    seg = torch.zeros(batch, g.tokens, dtype=torch.int64, device=device)
    seg[:, g.tokens // 2:] = 1
    if g.head == "qa":
        y = torch.randint(0, g.tokens, (2 * batch,), device=device, generator=gen)
    else:
        y = torch.randint(0, g.classes, (batch,), device=device, generator=gen)
    return torch.stack([tok, seg]), y


def make_executor(g, batch: int, dev):
    if g.kind == "vit":
        from paper_2102_03161_b200.vit import VitExecutor
        return VitExecutor(g, max_batch=batch, seed=17, device=dev)
    from paper_2102_03161_b200.bert import BertExecutor
    return BertExecutor(g, max_batch=batch, seed=17, device=dev)


def data_note(g) -> str:
    if g.kind == "vit":
        return ("synthetic (seeded N(0,1) images, uniform labels; random trunc-normal "
                "weights)")
    return ("synthetic (seeded uniform token ids, two segments, uniform "
            + ("span start/end labels" if g.head == "qa" else "class labels")
            + "; random trunc-normal weights)")


# ---- reference arm -------------------------------------------------------------
CPU_BATCH = {"vit-b16": 4, "vit-b16-cifar100": 4, "bert-base-384": 1, "bert-large-128": 2,
             "tiny-vit": 64}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_steps(cfg: str, steps: int, warmup: int, seconds: float = None):
    """fp32 CPU restatement of the train step (oracle/{vit,bert}_fp32.py,
    forward + backward + SGD) on all host cores over CPU_BATCH[cfg] samples
    per step: `warmup` untimed steps, then `steps` timed ones (or as many as
    fit in `seconds`).  Returns (per-step seconds, sample batch, threads)."""
    from oracle import bert_fp32, vit_fp32
    from paper_2102_03161_b200.configs import GEOMETRIES
    g = GEOMETRIES[cfg]
    b = CPU_BATCH[cfg]
    torch.set_num_threads(os.cpu_count() or 1)
    gen = torch.Generator().manual_seed(5)
    if g.kind == "vit":
        from paper_2102_03161_b200.vit import init_params
        params = init_params(g, seed=17)
        x, y = synthetic_inputs(g, b, gen, "cpu")
        one = lambda: vit_fp32.train_step(params, x, y, g, 0)[1]  # noqa: E731
    else:
        from paper_2102_03161_b200.bert import init_params
        params = init_params(g, seed=17)
        x, y = synthetic_inputs(g, b, gen, "cpu")
        lab = y.view(2, b) if g.head == "qa" else y
        one = lambda: bert_fp32.train_step(params, x[0], x[1], lab, g, 0)[1]  # noqa: E731

    def step():
        grads = one()
        with torch.no_grad():
            for k in params:
                params[k] -= 1e-3 * grads[k]

    for _ in range(max(1, warmup)):
        step()
    times, t_all = [], time.perf_counter()
    while True:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if seconds is None and len(times) >= steps:
            break
        if seconds is not None and time.perf_counter() - t_all >= seconds:
            break
    return times, b, torch.get_num_threads()


def cpu_baseline(cfg: str, seconds: float):
    times, b, cores = cpu_steps(cfg, 0, 1, seconds)
    el = sum(times)
    return {"value": round(len(times) * b / el, 3), "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{len(times)} steps x {b} samples of the {cfg} train step (fp32 "
                      f"PyTorch-CPU restatement, forward+backward+SGD) in {el:.1f}s"}


def reference_planner_time(cfg: str, gpus: int):
    """The reference's own CPU code path: its simulator (simulate_run,
    runner.cpp:94-305, built from /root/reference by `make oracle` into
    oracle/_ref/libeps_ref.so) on this config's scenario -- the control-plane
    time the decisions cost per run."""
    from paper_2102_03161_b200 import configs
    from paper_2102_03161_b200.capi import EpsApi
    lib = os.path.join(ROOT, "oracle/_ref/libeps_ref.so")
    if not os.path.exists(lib):
        return None
    api = EpsApi(lib, "epsref_")
    sc = api.scenario(configs.scenario(cfg, gpus))
    sc.simulate()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 0.5:
        rows, summ = sc.simulate()
        n += 1
    ms = 1000.0 * (time.perf_counter() - t0) / n
    return {"simulate_run_ms": round(ms, 3), "epochs": len(rows),
            "modeled_speedup": round(summ.get("speedup", float("nan")), 4),
            "source": "oracle/_ref/libeps_ref.so (reference sources, epsref_simulate_run)"}


def run_reference(args, world, rank):
    from paper_2102_03161_b200.configs import BATCH, GEOMETRIES
    if rank != 0:
        return  # the reference arm runs on rank 0 only
    cfg = args.config
    g = GEOMETRIES[cfg]
    times, b, cores = cpu_steps(cfg, args.steps, args.warmup)
    el = sum(times)
    v = len(times) * b / el
    out = {"impl": "reference", "metric": metric_of(cfg), "value": round(v, 3), "unit": UNIT,
           "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
           "ms_per_step": round(1000.0 * el / len(times), 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": data_note(g),
           "config": {"workload": f"{cfg}: {WORKLOADS[cfg][1]}; each step a bounded CPU sample "
                                  f"of {b} samples (fp32, forward+backward+SGD)",
                      "cpu_sample_batch": b, "global_batch": BATCH[cfg], "seq_len": g.tokens,
                      "parallelism": f"cpu x{cores} threads"},
           "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "port",
                            "cpu_model": cpu_model(),
                            "sample": f"{len(times)} timed steps x {b} samples in {el:.2f}s "
                                      f"(+{args.warmup} warm-up)"},
           "planner": reference_planner_time(cfg, max(1, args.gpus)),
           "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---- our arm -------------------------------------------------------------------
def main_ours(args, world, rank, local):
    from paper_2102_03161_b200 import LIB_PATH, configs, ops
    from paper_2102_03161_b200.capi import EpsApi
    from paper_2102_03161_b200.pipeline import EpsTransport, StagePlan, StageRunner, Transport
    from paper_2102_03161_b200.planner import Planner

    one_gpu = args.gloo_one_gpu
    dev = torch.device("cuda", 0 if one_gpu else local)
    torch.cuda.set_device(dev)
    nccl = None
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
            nccl = {"backend": "nccl", "version": ".".join(map(str, torch.cuda.nccl.version())),
                    "world_size": dist.get_world_size(),
                    "debug": os.environ.get("NCCL_DEBUG")}
    cfg = args.config
    g = configs.GEOMETRIES[cfg]
    batch = configs.BATCH[cfg]
    scen = configs.scenario(cfg, world)
    planner = Planner(EpsApi(LIB_PATH, "eps_"), scen)
    decisions = [planner.begin_epoch(e) for e in range(configs.EPOCHS[cfg])]
    plan0 = StagePlan.from_decision(decisions[0], g.layers)

    ex = make_executor(g, batch, dev)
    use_eps = world > 1 and not one_gpu and args.comm == "eps"
    transport = EpsTransport(rank, world) if use_eps else Transport(host_staged=one_gpu)
    if nccl is not None:
        nccl["data_path"] = ("eps_comm_* (libeps_b200.so, NCCL " +
                             str(transport.comm_version()) + ")" if use_eps
                             else "torch.distributed NCCL groups")
    runner = StageRunner(ex, rank, world, transport, peer=(args.p2p == "ipc"))
    runner.set_plan(plan0)
    pipe, stage = plan0.role(rank)
    gen = torch.Generator(device=dev).manual_seed(1234 + pipe)
    inputs, labels = synthetic_inputs(g, batch, gen, dev)
    stream = torch.cuda.current_stream()

    def step(x, cache_mode=0, cache_old=0, store=None, ids=None, lbls=None):
        loss = runner.iteration(x, labels if lbls is None else lbls, batch,
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

    energy_mj = []  # NVML energy reads at the two barriers of the metered (energy) run

    def timed(fn, steps, meter=False):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        if meter:
            energy_mj.append(clocks.energy_mj())
        s.record(stream)
        for _ in range(steps):
            fn()
        e.record(stream)
        barrier()
        if meter:
            energy_mj.append(clocks.energy_mj())
        return reduce(s.elapsed_time(e), dist.ReduceOp.MAX if world > 1 else None) / steps

    # ---- value: the epoch-0 (no-freeze) iteration, inputs resident in HBM ------
    for _ in range(args.warmup):
        step(inputs)
    clocks = ClockSampler(dev.index)
    clocks.start()
    n_launch0 = ops.launch_count()
    ms = timed(lambda: step(inputs), args.steps)
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
        step(inputs)
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
    # DRAM traffic per GEMM launch from the committed ncu --set full captures
    # (tools/gemm_traffic.py): the mean over forward, dgrad and wgrad launches
    # of this config, beside the algorithmic bytes of the same launches
    try:
        with open(os.path.join(ROOT, "profiles", "gemm_traffic.json")) as f:
            tr = json.load(f)
        t = tr["configs"][cfg]
        roofline["traffic"] = round(t["mean_dram_bytes_per_launch"])
        if "mean_algorithmic_bytes_per_launch" in t:
            roofline["traffic_algorithmic"] = round(t["mean_algorithmic_bytes_per_launch"])
        roofline["traffic_note"] = ("ncu dram__bytes_read+write per GEMM launch, mean over the "
                                    "profiled fwd / dgrad / wgrad launches "
                                    "(profiles/gemm_traffic.json)")
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
    h_inputs = inputs.cpu().pin_memory()
    h_labels = labels.cpu().pin_memory()
    first, last = stage == 0, stage == plan0.K - 1
    h2d = (h_inputs.numel() * h_inputs.element_size()
           + h_labels.numel() * h_labels.element_size()) * plan0.R
    d_in = [torch.empty_like(inputs) for _ in range(2)]
    d_lab = [torch.empty_like(labels) for _ in range(2)]
    h_loss = [torch.zeros(1, dtype=torch.float32).pin_memory() for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d_done, used, d2h_done = [ev(), ev()], [ev(), ev()], [ev(), ev()]
    state = {"i": 0, "losses": []}

    def prefetch(slot):
        copy_stream.wait_event(used[slot])
        with torch.cuda.stream(copy_stream):
            if first:
                d_in[slot].copy_(h_inputs, non_blocking=True)
            if last:
                d_lab[slot].copy_(h_labels, non_blocking=True)
            h2d_done[slot].record(copy_stream)

    prefetch(0)

    def e2e_step():
        i = state["i"]
        slot = i % 2
        stream.wait_event(h2d_done[slot])
        loss = step(d_in[slot], lbls=d_lab[slot])
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

    # ---- energy: board joules per step (NVML counter, every rank's GPU) ---------
    # The B200s run at their power limit, so throughput follows energy per
    # sample.  The counter updates too coarsely for a K-step window of a few
    # hundred ms, so this is its own ~2 s run of the step, placed after the
    # timed, instrumented and e2e runs so its heat does not reach them.
    energy = None
    if not args.no_energy:
        n_e = max(args.steps, int(2000.0 / ms) + 1)
        ms_e = timed(lambda: step(inputs), n_e, meter=True)
        if len(energy_mj) == 2 and None not in energy_mj:
            # (--gloo-one-gpu: every rank reads the same board)
            gpus = 1 if one_gpu else world
            ej = (energy_mj[1] - energy_mj[0]) / 1e3
            ej = ej if gpus == 1 else reduce(ej, dist.ReduceOp.SUM)
            energy = {"joules_per_step": round(ej / n_e, 3),
                      "samples_per_joule": round(plan0.R * batch * n_e / ej, 2),
                      "mean_w_per_gpu": round(ej / gpus / (ms_e * n_e / 1000.0), 1),
                      "steps": n_e, "ms_per_step": round(ms_e, 3),
                      "source": "NVML total energy counter at the barriers of a separate "
                                "~2 s run of the same step after the timed, instrumented "
                                "and e2e runs"}

    # ---- freeze schedule: the planner's per-epoch decisions on the device ------
    sched = None
    if not args.no_schedule:
        sched = freeze_schedule(runner, g, batch, decisions, inputs, step, timed, ms, dev)

    # ---- a K = 8 pipeline stage, emulated on this GPU ---------------------------
    emu = None
    if world == 1 and not args.no_stage_emulation and g.layers >= 8:
        emu = stage_emulation(ex, cfg, g, batch, inputs, labels, ms)

    del runner, ex
    if use_eps:
        transport.close()
    torch.cuda.empty_cache()

    # ---- the real epoch loop: freeze vs no-freeze, transitions included --------
    trainer = None
    if not args.no_trainer and g.kind == "vit" and not one_gpu:
        trainer = trainer_run(cfg, g, world, rank, dev, args.trainer_iters,
                              "eps" if use_eps else "torch")

    # the same loop with the host side in C++ (csrc/runtime/trainer.cpp, one GPU)
    trainer_native = None
    if not args.no_trainer and world == 1:
        trainer_native = trainer_run_native(cfg, g, args.trainer_iters)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args.cpu_seconds)

    if rank == 0:
        par = f"pipe{plan0.K}" + (f"xdp{plan0.R}" if plan0.R > 1 else "")
        out = {"metric": metric_of(cfg), "value": round(value, 2), "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
               "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
               "vs_baseline": None, "dtype": "bf16", "data": data_note(g),
               "config": {"workload": f"{cfg}: {WORKLOADS[cfg][1]}; no-freeze iteration "
                                      "(fwd+bwd+SGD) under the reference planner's epoch-0 plan",
                          "model": cfg, "global_batch": batch * plan0.R,
                          "seq_len": g.tokens, "parallelism": par,
                          "planner": {"K": plan0.K, "R": plan0.R, "M": plan0.M,
                                      "spans": [list(x) for x in plan0.spans]},
                          "l2": "inputs + activation working set (GBs) far exceed the 126 MB "
                                "L2 between iterations: no flush needed"},
               "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": 4 * plan0.R, "ms_per_step": round(e2e_ms, 3)},
               "gpu_launches": launches,
               "roofline": roofline,
               "kernels": kernels,
               "mfu": round(mfu, 4),
               "clocks": clock_rec,
               "energy": energy,
               "freeze_schedule": sched,
               "trainer_run": trainer,
               "trainer_run_native": trainer_native,
               "stage_emulation": emu,
               "nccl": nccl,
               "cpu_baseline": cpu}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def stage_emulation(ex, cfg, g, batch, inputs, labels, ms_whole):
    """Per-micro-batch forward + backward time of every stage of the
    reference planner's 1 x 8 epoch-0 plan (K = 8, M micro-batches of
    batch / M samples), each stage's sublayer span run on this one GPU with
    the same executor entry points a pipeline rank uses.  GPipe bound for the
    8-GPU iteration: (M + K - 1) x the slowest stage (schedule.cpp:56-116),
    P2P hand-off excluded (a 17-sample ViT cut is 5 MB: ~6 us at 900 GB/s)."""
    from paper_2102_03161_b200 import configs
    from paper_2102_03161_b200.capi import EpsApi
    from paper_2102_03161_b200 import LIB_PATH
    from paper_2102_03161_b200.pipeline import StagePlan, microbatch_offsets
    from paper_2102_03161_b200.planner import Planner
    d = Planner(EpsApi(LIB_PATH, "eps_"), configs.scenario(cfg, 8)).begin_epoch(0)
    plan = StagePlan.from_decision(d, g.layers)
    b = microbatch_offsets(batch, plan.M)[0][1]
    rows = []
    st = torch.cuda.current_stream()
    for s, (g0, g1) in enumerate(plan.spans):
        last = s == plan.K - 1

        def mb():
            ex.stage_forward(inputs if s == 0 else None, 0, b, g0, g1, 0, front=(s == 0))
            if last:
                ex.stage_head(labels, 0, b, batch)
            ex.stage_backward(0, b, g0, g1, 0, cut_out=not last)

        for _ in range(3):
            mb()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        for _ in range(10):
            mb()
        e.record(st)
        torch.cuda.synchronize()
        rows.append({"stage": s, "span": [g0, g1], "ms_per_microbatch": round(
            a.elapsed_time(e) / 10, 4)})
    ex.g32.zero_()
    slow = max(r["ms_per_microbatch"] for r in rows)
    t_iter = (plan.M + plan.K - 1) * slow
    return {"plan": {"K": plan.K, "M": plan.M, "micro_batch": b},
            "stages": rows, "slowest_stage_ms": slow,
            "gpipe_iteration_ms": round(t_iter, 3),
            "emulated_8gpu_samples_per_s": round(batch / (t_iter / 1000.0), 1),
            "whole_model_ms": round(ms_whole, 3),  # the full per-pipeline batch on one GPU
            "note": "single-GPU emulation of the 1x8 epoch-0 plan; not an 8-GPU measurement"}


def trainer_run(cfg, g, world, rank, dev, iters, comm="torch"):
    """The real epoch loop (paper_2102_03161_b200.trainer.Trainer): device
    gradient norms -> reference planner -> plan transition (weights, momentum,
    cache store) -> the epoch's iterations, for the freeze scenario and for
    the no-freeze baseline (runner.cpp:67-90); speedup = total no-freeze time
    / total freeze time, transitions included (runner.cpp:298)."""
    from paper_2102_03161_b200 import configs
    from paper_2102_03161_b200.trainer import Trainer
    out = {}
    for name, sc in (("freeze", configs.scenario(cfg, world)),
                     ("no_freeze", configs.no_freeze(configs.scenario(cfg, world)))):
        tr = Trainer(sc, g, iterations_per_epoch=iters, rank=rank, world=world, device=dev,
                     comm=comm)
        rows = tr.run()
        out[name] = {"total_s": round(sum(r.epoch_time_s + r.transition_time_s for r in rows), 4),
                     "epochs": [{"epoch": r.epoch, "l_frozen": r.l_frozen, "K": r.k, "R": r.r,
                                 "M": r.m, "cache": r.cache_enabled, "moved": r.cache_moved,
                                 "epoch_s": round(r.epoch_time_s, 4),
                                 "transition_s": round(r.transition_time_s, 4),
                                 "samples_per_s": round(r.throughput_sps, 1)} for r in rows]}
        del tr
        torch.cuda.empty_cache()
    out["speedup_vs_no_freeze"] = round(out["no_freeze"]["total_s"] / out["freeze"]["total_s"], 4)
    out["iterations_per_epoch"] = iters
    out["note"] = ("Trainer epochs with device gradient norms feeding the reference planner; "
                   "totals include set_plan transitions and cache boundary moves")
    return out


def trainer_run_native(cfg, g, iters):
    """trainer_run with the epoch loop in C++ (eps_trainer_*: planner, shards,
    AutoCache modes, device norms; csrc/runtime/trainer.cpp) on one GPU."""
    from paper_2102_03161_b200 import configs
    from paper_2102_03161_b200.native_trainer import NativeTrainer
    out = {}
    for name, sc in (("freeze", configs.scenario(cfg, 1)),
                     ("no_freeze", configs.no_freeze(configs.scenario(cfg, 1)))):
        tr = NativeTrainer(sc, g, iterations_per_epoch=iters)
        rows = tr.run(int(sc["training"]["epochs"]))
        tr.close()
        out[name] = {"total_s": round(sum(r.epoch_time_s for r in rows), 4),
                     "epochs": [{"epoch": r.epoch, "l_frozen": r.l_frozen, "cache": r.cache_enabled,
                                 "moved": r.cache_moved, "epoch_s": round(r.epoch_time_s, 4),
                                 "loss": round(r.mean_loss, 4),
                                 "samples_per_s": round(r.throughput_sps, 1)} for r in rows]}
        torch.cuda.empty_cache()
    out["speedup_vs_no_freeze"] = round(out["no_freeze"]["total_s"] / out["freeze"]["total_s"], 4)
    out["iterations_per_epoch"] = iters
    out["note"] = ("native C++ epoch loop (eps_trainer_run_epoch), device gradient norms feeding "
                   "the reference planner; seeded synthetic data and init inside the library")
    return out


def freeze_schedule(runner, g, batch, decisions, inputs, step, timed, ms0, dev):
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
                step(inputs, 2, 0, store, ids)
            fn = lambda: step(inputs, mode, old, store if mode else None,  # noqa: E731
                              ids if mode else None)
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
            "note": "steady-state replay: per-epoch decisions from the reference planner (its "
                    "synthetic norms), each executed on the device (K-stage pipelines x R "
                    "replicas); transitions excluded -- see trainer_run for the real loop"}


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    if world > 1 and not args.gloo_one_gpu:
        # rank / NVLink / NVLS evidence in the log (NCCL's INIT lines)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    main_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
