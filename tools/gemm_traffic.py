"""Per-launch DRAM traffic of the profiled block GEMMs (ncu --set full report)
-> profiles/gemm_traffic.json, which bench.py reports as roofline.traffic.

    python tools/gemm_traffic.py gpurun_out/prof_gemm.ncu-rep profiles/gemm_traffic.json
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    launches = []
    for r in rows[2:]:
        rd = hdr.index("dram__bytes_read.sum")
        wr = hdr.index("dram__bytes_write.sum")
        tb = float(r[rd].replace(",", "")) * scale[units[rd]] + \
            float(r[wr].replace(",", "")) * scale[units[wr]]
        launches.append({"kernel": r[hdr.index("Kernel Name")].split("(")[0],
                         "grid": r[hdr.index("Grid Size")], "dram_bytes": tb})
    res = {"source": rep, "launches": launches,
           "mean_dram_bytes_per_launch": sum(l["dram_bytes"] for l in launches) / len(launches)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res)[:400])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
