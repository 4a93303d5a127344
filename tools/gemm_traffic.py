"""Per-launch DRAM traffic of profiled block GEMMs (ncu --set full reports)
beside each launch's algorithmic bytes -> profiles/gemm_traffic.json, which
bench.py reports as roofline.traffic (mean over the launches).

    python tools/gemm_traffic.py OUT.json CFG REP:ROLE,ROLE,... [REP:ROLE,...]

ROLE names one launch of the report, in capture order, from SHAPES (ViT-B/16
b400: R = 78,800 token rows).  Algorithmic bytes = operands read once +
outputs written once (+ aux inputs / second outputs of fused epilogues);
fp32 weight-gradient accumulators count one read + one write (the split-K
TMA reduce-add).
"""
import csv
import io
import json
import subprocess
import sys

R = 400 * 197
D, F = 768, 3072
BF, F32 = 2, 4
# role: (M, N, K, bytes)
SHAPES = {
    "fwd_qkv": (R, 3 * D, D, BF * (R * D + 3 * D * D + R * 3 * D)),
    "fwd_proj_resid": (R, D, D, BF * (R * D + D * D + 2 * R * D)),
    "fwd_fc1_gelu2": (R, F, D, BF * (R * D + F * D + 2 * R * F)),
    "fwd_fc2_resid": (R, D, F, BF * (R * F + F * D + 2 * R * D)),
    "wgrad_fc2": (D, F, R, BF * (R * D + R * F) + 2 * F32 * D * F),
    "dgrad_fc2_mul": (R, F, D, BF * (R * D + F * D + 2 * R * F)),
    "wgrad_fc1": (F, D, R, BF * (R * F + R * D) + 2 * F32 * D * F),
    "dgrad_fc1": (R, D, F, BF * (R * F + F * D + R * D)),
    "wgrad_proj": (D, D, R, BF * 2 * R * D + 2 * F32 * D * D),
    "dgrad_proj_rowdot": (R, D, D, BF * (R * D + D * D + 2 * R * D) + F32 * R * 12),
    "wgrad_qkv": (3 * D, D, R, BF * (R * 3 * D + R * D) + 2 * F32 * 3 * D * D),
    "dgrad_qkv": (R, D, 3 * D, BF * (R * 3 * D + 3 * D * D + R * D)),
}
METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6,
         "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9, "%": 1}


def read(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        v = {}
        for m in METRICS:
            cols = [i for i, h in enumerate(hdr) if h == m]
            if cols:
                i = cols[0]
                v[m] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
        v["kernel"] = r[hdr.index("Kernel Name")].split("(")[0]
        out.append(v)
    return out


def main(out_path, cfg, specs):
    launches = []
    for spec in specs:
        rep, roles = spec.split(":")
        for v, role in zip(read(rep), roles.split(",")):
            M, N, K, alg = SHAPES[role]
            dram = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
            t = v["gpu__time_duration.sum"]
            launches.append({"role": role, "kernel": v["kernel"], "M": M, "N": N, "K": K,
                             "dram_bytes": dram, "algorithmic_bytes": alg,
                             "traffic_over_algorithmic": round(dram / alg, 3),
                             "ncu_us": round(t * 1e6, 1),
                             "ncu_tflops": round(2.0 * M * N * K / t / 1e12, 1),
                             "tensor_pipe_active_pct": round(v.get(METRICS[3], float("nan")), 1)})
    n = len(launches)
    res = {"configs": {cfg: {
        "source": specs, "launches": launches,
        "mean_dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) / n,
        "mean_algorithmic_bytes_per_launch": sum(x["algorithmic_bytes"] for x in launches) / n,
        "note": "ncu --set full --clock-control none (serialised, cold L2 per replay); "
                "layer-1 forward + layer-11 backward GEMMs of one ViT-B/16 b400 step"}}}
    try:
        old = json.load(open(out_path))
        for k, v in old.get("configs", {}).items():
            res["configs"].setdefault(k, v)
    except (OSError, ValueError):
        pass
    json.dump(res, open(out_path, "w"), indent=1)
    for x in launches:
        print(x)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3:])
