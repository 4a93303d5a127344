"""Summarise an ncu source page (per-SASS-instruction warp-stall samples).

    ncu -i REP --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv [top_n]

Prints the stall-reason totals over the kernel and the top_n instructions
by sample count with their dominant reasons."""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]
    tot = {h: sum(float(r[idx[h]] or 0) for r in body) for h in reasons}
    allsum = sum(tot.values())
    print("kernel:", rows[0][1][:100])
    print("total samples", int(allsum))
    for h, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
        print(f"  {h:28s} {v / allsum:6.1%}")
    body.sort(key=lambda r: -float(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
    print(f"top {top} instructions:")
    for r in body[:top]:
        n = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        rs = sorted(((float(r[idx[h]] or 0), h[6:]) for h in reasons), reverse=True)[:3]
        print(f"{n / allsum:6.2%} {r[idx['Address']][-5:]} {r[idx['Source']].strip()[:60]:60s} "
              + " ".join(f"{h}:{v / max(n, 1):.0%}" for v, h in rs if v > 0))


if __name__ == "__main__":
    main()
