"""Per-source-line warp-stall samples from `ncu --page source --csv --print-source cuda,sass` output."""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    path, hdr, out = None, None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and r[0].isdigit() and len(r) >= 5:
            try:
                v = float(r[4])
            except ValueError:
                continue
            if v > 0:
                out.append((v, f"{path}:{r[0]}", r[1].strip()[:90]))
    tot = sum(o[0] for o in out) or 1
    for v, where, src in sorted(out, reverse=True)[:top]:
        print(f"{v / tot:6.1%} {where:28s} {src}")


if __name__ == "__main__":
    main()
