# full default bench (config 5 + e2e + solve + cpu + secondary); reference arm; cfg4 dense mode; ncu of dense hv
set -x
mkdir -p gpurun_out/r2f
timeout 1500 python bench.py > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err; echo bench_exit=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2f/bench_ref.json 2> gpurun_out/r2f/bench_ref.err; echo ref_exit=$?
OTB_HV_DENSE=1 timeout 900 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --steps 5 > gpurun_out/r2f/bench_cfg4_dense.json 2>gpurun_out/r2f/bench_cfg4_dense.err; echo c4d_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(hv_wc|eval|test_c)" --launch-skip 40 -c 3 -o gpurun_out/r2f/k5 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/r2f/ncu5.log 2>&1; echo ncu5_exit=$?
for f in gpurun_out/r2f/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
rm -f gpurun_out/r2f/*.ncu-rep
