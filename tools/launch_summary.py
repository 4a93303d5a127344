"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per kernel family, launches, total device time and share of the total.

    python tools/launch_summary.py gpurun_out/launches.csv [> profiles/....md]
"""
import csv
import re
import sys
from collections import defaultdict


def family(name: str) -> str:
    m = re.match(r"(?:void )?(?:[\w:]+::)?(\w+)", name)
    base = m.group(1) if m else name
    t = re.search(r"<([^<>]*)>", name)
    if base == "gemm_tc_kernel" and t:
        base += "<" + t.group(1) + ">"
    return base


def main(path):
    agg = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        rows = [r for r in csv.DictReader(l for l in f if l.startswith('"'))]
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1.0)
        k = family(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ns * scale
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.1f}% |")
    print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | 100% |")


if __name__ == "__main__":
    main(sys.argv[1])
