# ncu source-level capture of the config-5 dense passes (per-instruction executed counts + stall samples)
set -x
mkdir -p gpurun_out/r2q
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(eval|test_b|test_c|test_a|sparsify)" --launch-skip 5 -c 5 -o gpurun_out/r2q/dense5 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 1 --warmup 3 > gpurun_out/r2q/ncu5d.log 2>&1; echo ncud_exit=$?
for f in gpurun_out/r2q/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
ls -la gpurun_out/r2q
rm -f gpurun_out/r2q/*.ncu-rep
