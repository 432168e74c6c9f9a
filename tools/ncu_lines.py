"""Per-source-line executed instructions of an ncu report (cuda,sass view):
the hottest CUDA lines with their share of the kernel's instructions.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur_file, per = None, collections.Counter()
    texts = {}
    hdr = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or len(row) < len(hdr) or not row[0].isdigit():
            continue
        ie = hdr.index("Instructions Executed")
        try:
            n = int(row[ie] or 0)
        except ValueError:
            continue
        key = (cur_file, int(row[0]))
        per[key] += n
        texts.setdefault(key, row[1].strip()[:90])
    tot = sum(per.values())
    print(f"total {tot / 1e6:.3f}M")
    for (f, ln), n in per.most_common(top):
        print(f"{100 * n / tot:5.1f}% {n / 1e6:7.3f}M {f}:{ln}  {texts[(f, ln)]}")


if __name__ == "__main__":
    main()
