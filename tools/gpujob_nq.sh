# config 4 dense-P_rho hess_apply: window width (NQ) 8 (W = 2, 148 SMs, register spills) vs 4 and 6
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
for NQ in 8 4 6; do
  OTB_HV_NQ=$NQ timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench4_nq$NQ.json 2>gpurun_out/$T/bench4_nq$NQ.err; echo nq$NQ=$?
done
python tools/bench_brief.py gpurun_out/$T/bench4_nq*.json
