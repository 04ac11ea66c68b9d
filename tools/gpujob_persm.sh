# two CTAs per SM for the dense passes (OTB_DENSE_CTAS_PER_SM=2) against one: gpu suite and step benches
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
OTB_DENSE_CTAS_PER_SM=2 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_persm2.log 2>&1; echo all_exit=$?; tail -3 gpurun_out/$T/pytest_persm2.log
for P in 1 2; do
  OTB_DENSE_CTAS_PER_SM=$P timeout 600 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench5_p$P.json 2>gpurun_out/$T/bench5_p$P.err; echo b5_$P=$?
  OTB_DENSE_CTAS_PER_SM=$P timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench4_p$P.json 2>gpurun_out/$T/bench4_p$P.err; echo b4_$P=$?
  OTB_DENSE_CTAS_PER_SM=$P timeout 600 python bench.py --config 3 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench3_p$P.json 2>gpurun_out/$T/bench3_p$P.err; echo b3_$P=$?
done
python tools/bench_brief.py gpurun_out/$T/bench*_p*.json
