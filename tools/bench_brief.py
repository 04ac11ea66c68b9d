"""One line per bench JSON: value and per-kernel (us per launch, fraction of peak).
    python tools/bench_brief.py gpurun_out/TAG/bench5.json ..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        pk = d["roofline"]["per_kernel"]
        print(f, round(d["value"], 3), {k: (round(v["us_per_launch"]), round(v.get("frac", 0), 3)) for k, v in pk.items()})
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
