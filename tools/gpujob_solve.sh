# gpu suite + solve-to-tol lines on configs 1-3 and 5 (the half of BASELINE's metric the step bench does not cover)
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_all.log 2>&1; echo all_exit=$?; tail -3 gpurun_out/$T/pytest_all.log
timeout 900 python bench.py --no-cpu --e2e-steps 0 --secondary "2,3" --steps 2 > gpurun_out/$T/bench5.json 2>gpurun_out/$T/bench5.err; echo b5_exit=$?
python - <<PY
import json
d=json.loads(open("gpurun_out/$T/bench5.json").read().strip().splitlines()[-1])
print("cfg5 step", d["value"], "solve", d.get("solve"))
for k,v in (d.get("secondary") or {}).items(): print(k, v["value"], v.get("solve"))
PY
