# ring-depth experiment: config-5 step bench with the dense ring capped at 3/5/8 stages
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
for NSG in 3 5 8; do
  OTB_DENSE_NSTAGE=$NSG timeout 600 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/$T/bench5_ns$NSG.json 2>gpurun_out/$T/bench5_ns$NSG.err; echo ns${NSG}_exit=$?
done
python tools/bench_brief.py gpurun_out/$T/bench5_ns*.json
