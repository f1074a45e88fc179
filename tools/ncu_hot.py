"""Summarise an ncu source page (SASS) export: top instructions by warp-stall samples.

usage: ncu -i rep --page source --csv --print-source sass [--launch-skip N --launch-count 1] > x.csv
       python tools/ncu_hot.py x.csv [top]
"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    hdr = rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ei = hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    total = sum(float(r[si] or 0) for r in body)
    print(f"total samples {total:.0f}, instructions {len(body)}")
    agg = {}
    for r in body:
        for i in stall_cols:
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i] or 0)
    print("stall mix:", ", ".join(f"{k[6:]}={v / total:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    order = sorted(range(len(body)), key=lambda j: -float(body[j][si] or 0))
    for j in order[:top]:
        r = body[j]
        st = sorted(((hdr[i][6:], float(r[i] or 0)) for i in stall_cols), key=lambda x: -x[1])[:2]
        print(f"{j:6d} {float(r[si]) / total:6.2%} ex={r[ei]:>10} {r[1].strip()[:60]:60s} {st}")


if __name__ == "__main__":
    main()
