"""Summarise an `ncu --set full` report into profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep|RAW.csv OUT_DIR [config_key]

(RAW.csv = `ncu -i REPORT --page raw --csv` made on the GPU box when the
report itself is too large to copy back.)

Writes OUT_DIR/ncu_full_summary.csv (one row per captured launch: duration,
DRAM bytes read/written, achieved DRAM GB/s, issue-slot use, pipe shares,
registers, top stall reasons) and merges the per-launch DRAM traffic of each
kernel class into profiles/traffic.json under `config_key` (default cfg2) —
the `traffic` field of bench.py's roofline object.
"""

import csv
import io
import json
import os
import subprocess
import sys

CLASS = {"k_cg_fused": "cg_fused", "k_eval": "eval", "k_sparsify_dense": "sparsify", "k_sparsify": "sparsify",
         "k_test_a": "test_a", "k_hv_wcd": "hess_apply",
         "k_test_b": "test_b", "k_test_c": "test_c", "k_hv_grp": "hess_apply", "k_hv_wc": "hess_apply", "k_warm_zeta": "warm_zeta",
         "k_warm_gamma": "warm_gamma"}

KEYS = [("gpu__time_duration.sum", "duration_us", 1e-3),
        ("dram__bytes_read.sum", "dram_read_MB", None),
        ("dram__bytes_write.sum", "dram_write_MB", None),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_pct", 1),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_pipe_pct", 1),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_pct", 1),
        ("smsp__inst_executed.sum", "warp_instructions", 1),
        ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1),
        ("launch__registers_per_thread", "registers", 1),
        ("launch__grid_size", "grid", 1),
        ("launch__block_size", "block", 1)]


def to_mb(v, unit):
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1e-6)
    return v * scale


def main():
    rep, out_dir = sys.argv[1], sys.argv[2]
    key = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
    if rep.endswith(".csv"):
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name-base", "function"],
                             capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out_rows = []
    traffic = {}
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        base = name.split("<")[0].split("(")[0].strip().split(" ")[-1]
        row = {"id": d.get("ID"), "kernel": name[:60]}
        for k, label, scale in KEYS:
            v = d.get(k, "")
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                row[label] = ""
                continue
            if label.endswith("_MB"):
                x = to_mb(x, u.get(k, ""))
            elif label == "duration_us":
                x = x * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                         "s": 1e6, "second": 1e6}.get(u.get(k, ""), 1e-3)
            row[label] = round(x, 3)
        try:
            row["dram_GBps"] = round((row["dram_read_MB"] + row["dram_write_MB"]) * 1e-3 / (row["duration_us"] * 1e-6), 1)
        except (TypeError, ZeroDivisionError):
            row["dram_GBps"] = ""
        stalls = [(float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                  for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not k.endswith("not_issued") and v.replace(",", "").replace(".", "").isdigit()]
        tot = sum(s for s, _ in stalls) or 1.0
        row["top_stalls"] = "; ".join(f"{k} {100 * s / tot:.0f}%" for s, k in sorted(stalls, reverse=True)[:3])
        out_rows.append(row)
        cls = CLASS.get(base)
        if cls and row.get("dram_read_MB") != "":
            traffic.setdefault(cls, []).append((row["dram_read_MB"] + row["dram_write_MB"]) * 1e6)
    os.makedirs(out_dir, exist_ok=True)
    fields = ["id", "kernel", "duration_us", "dram_read_MB", "dram_write_MB", "dram_GBps"] + \
        [lab for _, lab, _ in KEYS if lab not in ("duration_us", "dram_read_MB", "dram_write_MB")] + ["top_stalls"]
    out_name = os.environ.get("NCU_SUMMARY_NAME", "ncu_full_summary.csv")
    with open(os.path.join(out_dir, out_name), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=fields)
        w.writeheader()
        for row in out_rows:
            w.writerow({k: row.get(k, "") for k in fields})
    tpath = os.path.join(os.path.dirname(os.path.abspath(out_dir)), "traffic.json")
    allt = json.load(open(tpath)) if os.path.exists(tpath) else {}
    allt.setdefault(key, {})
    for cls, vals in traffic.items():
        allt[key][cls] = sum(vals) / len(vals)
    json.dump(allt, open(tpath, "w"), indent=1, sort_keys=True)
    for row in out_rows:
        print(row)


if __name__ == "__main__":
    main()
