"""Summarise an ncu launch-list CSV (gpu__time_duration + dram bytes per launch):
per-launch table of the first solve's kernels and per half-step totals.

  python tools/launch_summary.py gpurun_out/launches_c2.csv [N]
"""
import collections
import csv
import re
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    per = collections.OrderedDict()
    for r in data:
        d = per.setdefault(r[ii], {"k": r[ki], "g": r[gi] if gi is not None else ""})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(per.values())


def short(k):
    m = re.search(r"(hm2?_\w+kernel)<(\d+), (\d+)", k)
    return f"{m.group(1)}<LPL={m.group(2)},V={m.group(3)}>" if m else k.split("(")[0][:34]


def main():
    seq = load(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else len(seq)
    tot = sum(p["gpu__time_duration.sum"] for p in seq[:n])
    print("| kernel | grid | us | MB DRAM |\n|---|---|---|---|")
    for p in seq[:n]:
        mb = (p.get("dram__bytes_read.sum", 0) + p.get("dram__bytes_write.sum", 0)) / 1e6
        print(f"| `{short(p['k'])}` | {p['g']} | {p['gpu__time_duration.sum'] / 1e3:.1f} | {mb:.1f} |")
    print(f"| total | | {tot / 1e3:.1f} | |")
    cls = collections.defaultdict(float)
    for p in seq[:n]:
        cls[short(p["k"]).split("<")[0]] += p["gpu__time_duration.sum"] / 1e3
    print("\n| class | us | share |\n|---|---|---|")
    for k, v in sorted(cls.items(), key=lambda x: -x[1]):
        print(f"| {k} | {v:.1f} | {v / (tot / 1e3):.3f} |")


if __name__ == "__main__":
    main()
