# PCG tests, whole suite; ring-depth (gamma in L1) experiment; ncu of the dense hess_apply and eval
set -x
mkdir -p gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pcg" > gpurun_out/r2g/pytest_pcg.log 2>&1; echo pcg_exit=$?; tail -5 gpurun_out/r2g/pytest_pcg.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2g/pytest_all.log 2>&1; echo all_exit=$?; tail -5 gpurun_out/r2g/pytest_all.log
for ns in 4 5; do
  OTB_DENSE_NSTAGE=$ns timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary 2,3 --steps 3 > gpurun_out/r2g/bench_ns$ns.json 2>gpurun_out/r2g/bench_ns$ns.err; echo ns${ns}_exit=$?
done
timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary 2,3 --steps 3 > gpurun_out/r2g/bench_ns8.json 2>gpurun_out/r2g/bench_ns8.err; echo ns8_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_hv_wc" --launch-skip 50 -c 2 -o gpurun_out/r2g/hv5 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/r2g/ncu5.log 2>&1; echo ncuhv_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(eval|test_c|test_a|sparsify)" --launch-skip 4 -c 4 -o gpurun_out/r2g/dense5 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/r2g/ncu5d.log 2>&1; echo ncud_exit=$?
for f in gpurun_out/r2g/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
rm -f gpurun_out/r2g/*.ncu-rep
