"""Key metrics of an `ncu --set full` report, one row per profiled launch.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("duration us", "gpu__time_duration.sum"),
    ("DRAM read MB", "dram__bytes_read.sum"),
    ("DRAM write MB", "dram__bytes_write.sum"),
    ("DRAM % peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor pipe % active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs/thread", "launch__registers_per_thread"),
    ("grid", "Grid Size"),
    ("block", "Block Size"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "")
        vals = []
        for _, key in METRICS:
            if key not in hdr:
                vals.append("-")
                continue
            i = hdr.index(key)
            v, u = r[i], units[i]
            if u in ("byte", "Kbyte", "Mbyte", "Gbyte"):
                f = float(v.replace(",", "")) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1,
                                                  "Gbyte": 1e3}[u]
                v = f"{f:.1f}"
            elif u in ("nsecond", "usecond", "msecond"):
                f = float(v.replace(",", "")) * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}[u]
                v = f"{f:.1f}"
            vals.append(v)
        print(f"| `{short}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
