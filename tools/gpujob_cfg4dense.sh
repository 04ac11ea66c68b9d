# config 4 (37% kept): dense P_rho forced vs the bitmap runs, with the producer-free dense kernel
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
for D in 0 1; do
  OTB_HV_DENSE=$D timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench4_d$D.json 2>gpurun_out/$T/bench4_d$D.err; echo b4_$D=$?
done
OTB_HV_DENSE=1 timeout 600 python bench.py --config 3 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench3_d1.json 2>gpurun_out/$T/bench3_d1.err; echo b3_1=$?
python tools/bench_brief.py gpurun_out/$T/bench4_d*.json gpurun_out/$T/bench3_d1.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/$T/smoke.log
