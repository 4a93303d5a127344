"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report.

    python tools/ncu_hot.py report.ncu-rep [kernel-substring] [top]
"""
import csv
import io
import subprocess
import sys


def main(path, kern="", top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    blocks, cur = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = [line.split(",", 1)[1], []]
            blocks.append(cur)
        elif cur is not None:
            cur[1].append(line)
    for name, lines in blocks:
        if kern not in name:
            continue
        rows = list(csv.reader(io.StringIO("\n".join(lines))))
        hdr = rows[0]
        isamp, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        body = rows[1:]
        tot = sum(float(r[isamp] or 0) for r in body)
        totx = sum(float(r[iex] or 0) for r in body)
        print(f"== {name[:100]}  samples={tot:.0f} warp-instr={totx:.0f}")
        for i, r in sorted(enumerate(body), key=lambda ir: -float(ir[1][isamp] or 0))[:top]:
            print(f"{i:5d} {float(r[isamp] or 0) / tot * 100:5.1f}%  ex={r[iex]:>9}  {r[1].strip()[:90]}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "",
         int(sys.argv[3]) if len(sys.argv) > 3 else 40)
