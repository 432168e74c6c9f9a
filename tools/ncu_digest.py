"""Digest of an ncu --set full report: headline metrics and the per-opcode
executed-instruction mix / stall samples from the SASS source page.

  python tools/ncu_digest.py gpurun_out/x.ncu-rep [launch-index]   (reports with several kernels)
"""
import collections
import csv
import io
import subprocess
import sys

HEAD = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + KSEL, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def sass(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + KSEL,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    body = []
    for r in rows[2:]:                      # the first kernel's block only
        if r and r[0] == "Kernel Name":
            break
        body.append(r)
    return hdr, body


KSEL = []


def main():
    rep = sys.argv[1]
    if len(sys.argv) > 2:
        KSEL.extend(["--print-kernel-base", "function", "--launch-skip", sys.argv[2], "--launch-count", "1"])
    r = raw(rep)
    print(f"# {r.get('Kernel Name', ('?', ''))[0][:160]}\n")
    print("| metric | unit | value |\n|---|---|---|")
    for h in HEAD:
        if h in r:
            print(f"| `{h}` | {r[h][1]} | {r[h][0]} |")
    stalls = sorted(((float(v[0].replace(',', '')), h) for h, v in r.items()
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")
                     and v[0] not in ("", "n/a")), reverse=True)[:8]
    for v, h in stalls:
        print(f"| `{h}` | | {v:.3f} |")
    hdr, data = sass(rep)
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    sm = hdr.index("Warp Stall Sampling (All Samples)")
    ops, smp = collections.Counter(), collections.Counter()
    for row in data:
        if len(row) <= max(ie, src, sm):
            continue
        t = row[src].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op] += int(row[ie] or 0)
        smp[op] += int(row[sm] or 0)
    tot, tots = sum(ops.values()), max(1, sum(smp.values()))
    print("\n```\nopcode                        executed   share  stall-samples")
    for op, n in ops.most_common(30):
        print(f"{op:28s} {n / 1e6:9.3f}M {100 * n / tot:6.1f}%  {100 * smp[op] / tots:6.1f}%")
    print(f"total {tot / 1e6:.3f}M\n```")


if __name__ == "__main__":
    main()
