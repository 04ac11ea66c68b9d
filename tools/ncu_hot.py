"""Summarise an ncu report: headline metrics and the hottest source lines.

    python tools/ncu_hot.py gpurun_out/x.ncu-rep 'k_sparsify' [top]

Reads the report with `ncu -i` (available in this container, no GPU needed)
and prints, for the first launch matching the regex: duration, issue-slot
use, pipe utilisation, instructions per processed element (when `elements`
is passed as argv[4]) and the source lines with the most executed
instructions / stall samples.
"""

import csv
import io
import subprocess
import sys


def ncu(*args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    elems = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
    raw = ncu("-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{kern}", "--launch-count", "1")
    hdr, vals = raw[0], raw[2]
    d = dict(zip(hdr, vals))
    keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "smsp__warps_eligible.avg.per_cycle_active"]
    print(d.get("Kernel Name", "?")[:80])
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    if elems and "smsp__inst_executed.sum" in d:
        print(f"  thread-instructions per element: {float(d['smsp__inst_executed.sum'].replace(',', '')) * 32 / elems:.1f}")
    rows = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name", f"regex:{kern}",
               "--launch-count", "1")
    out, fname = [], "?"
    for r in rows:
        if r and r[0] == "File Name":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 8 or r[0] == "Line No" or not r[0]:
            continue
        try:
            ie, ss = float(r[7] or 0), float(r[4] or 0)
        except ValueError:
            continue
        if ie > 0 or ss > 0:
            out.append((ie, ss, fname, r[0], r[1].strip()[:90]))
    tot = sum(o[0] for o in out) or 1.0
    tots = sum(o[1] for o in out) or 1.0
    for o in sorted(out, reverse=True)[:top]:
        print(f"{o[0] / tot * 100:5.1f}% inst {o[1] / tots * 100:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main()
