"""Attribute ncu warp-stall samples to CUDA source lines.

    nvdisasm -g KERNEL.cubin > all.dis    (the object the report was taken from)
    ncu -i REP --page source --csv --print-source sass > src.csv
    python tools/ncu_lines.py all.dis MANGLED_KERNEL src.csv [FILE_SUBSTR] [top]

The SASS offsets of the source page are mapped to the innermost line of
FILE_SUBSTR (default attention_tc.cu) that nvdisasm's line table gives them;
prints the top lines by sample share with their two main stall reasons."""
import csv
import re
import sys
from collections import Counter, defaultdict


def main():
    dis, kern, src = sys.argv[1:4]
    fsub = sys.argv[4] if len(sys.argv) > 4 else "attention_tc.cu"
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    off2line, cur, on = {}, None, False
    for line in open(dis):
        if line.startswith("//") and ".text." in line:
            on = (".text." + kern) in line and line.split(".text.")[1].split()[0] == kern
            continue
        if not on:
            continue
        m = re.search(re.escape(fsub) + r'", line (\d+)', line)
        if m:
            cur = int(m.group(1))
        m2 = re.search(r"/\*([0-9a-f]{4,5})\*/", line)
        if m2 and cur:
            off2line[int(m2.group(1), 16)] = cur
    rows = list(csv.reader(open(src)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
    base = int(body[0][0], 16)
    tot, per, why = 0.0, Counter(), defaultdict(Counter)
    for r in body:
        n = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        tot += n
        ln = off2line.get(int(r[0], 16) - base)
        per[ln] += n
        for h in reasons:
            why[ln][h[6:]] += float(r[idx[h]] or 0)
    for ln, n in per.most_common(top):
        rs = " ".join(f"{h}:{v / max(n, 1):.0%}" for h, v in why[ln].most_common(2))
        print(f"{n / tot:6.2%} line {ln}  {rs}")


if __name__ == "__main__":
    main()
