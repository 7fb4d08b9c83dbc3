"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel: share of device time per fit."""
import collections
import csv
import re
import sys

UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def summarise(path, fits, title):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    H, data = rows[hdr], rows[hdr + 1:]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        ms = float(r[vi].replace(",", "")) * UNIT[r[ui]]
        name = r[ki]
        short = re.sub(r"\(.*", "", name)
        if "cub" in name:
            m = re.search(r"Policy1000, 0, ([^,]+), ([^,]+),", name)
            short = "cub radix sort " + (f"{m.group(1)}->{m.group(2)}" if m else name[:60])
        tot[short] += ms
        cnt[short] += 1
    s = sum(tot.values())
    out = [f"# {title}", "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)",
           f"# {len(data)} launches over {fits} fits; device time per fit {s / fits:.2f} ms",
           "share%    ms/fit  launches/fit  kernel"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"{100 * v / s:6.2f} {v / fits:9.3f} {cnt[k] / fits:11.1f}   {k}")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]), sys.argv[3]), end="")
