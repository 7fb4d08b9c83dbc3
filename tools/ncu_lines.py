"""Aggregate ncu warp-stall samples by CUDA source line (ncu -i rep --page source --csv --print-source cuda,sass)."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    cur_file, cur_line, cur_src = "?", "?", ""
    agg, src = collections.Counter(), {}
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur_line, cur_src = r[0], r[1]
        try:
            w = float(r[4] or 0)
        except ValueError:
            continue
        key = (cur_file, int(cur_line) if cur_line.isdigit() else 0)
        agg[key] += w
        src[key] = cur_src
    tot = sum(agg.values())
    print(f"total samples {tot:.0f}")
    for k, v in agg.most_common(top):
        print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]}  {src[k].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
