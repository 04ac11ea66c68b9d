# hess_apply window width sweep at config 4 (OTB_HV_NQ), dense and bitmap P_rho
T=${1:-nq4}
mkdir -p gpurun_out/$T
for nq in 8 6 4 3 2; do
  for hd in 1 0; do
  OTB_HV_DENSE=$hd OTB_HV_NQ=$nq OTB_LIB=$PWD/_exp/nodefer/libotb.so timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/nq${nq}_d$hd.json 2>gpurun_out/$T/nq${nq}_d$hd.err || tail -3 gpurun_out/$T/nq${nq}_d$hd.err
  echo "nq=$nq dense=$hd"; python tools/bench_brief.py gpurun_out/$T/nq${nq}_d$hd.json
  done
done
