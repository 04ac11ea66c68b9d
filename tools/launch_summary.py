"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py gpurun_out/r1/launches.csv > profiles/r1/launch_summary.txt
"""
import csv
import sys
from collections import defaultdict


def main():
    rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
    rd = csv.DictReader(rows)
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        name = r["Kernel Name"]
        name = name.split("(")[0].replace("void ", "")
        tot[name] += us
        cnt[name] += 1
    total = sum(tot.values())
    print("ncu launch list of `bench.py --steps 2 --warmup 3 --no-solve --no-cpu` (cold-cache, serialised; shares, "
          "not absolutes)")
    print(f"launches {sum(cnt.values())}, total {total:.1f} us")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:30]:
        print(f"{v:10.1f} us {100 * v / total:5.1f}% {cnt[k]:5d}x  {k[:60]}")


if __name__ == "__main__":
    main()
