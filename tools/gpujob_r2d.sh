# st.async cluster exchanges (dense passes + hess_apply), dense cl choice; suite + cfg4/5 bench
set -x
mkdir -p gpurun_out/r2d
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2d/pytest_all.log 2>&1; echo all_exit=$?; tail -15 gpurun_out/r2d/pytest_all.log
timeout 900 python bench.py --config 5 --no-cpu --no-solve --steps 3 --warmup 3 > gpurun_out/r2d/bench_cfg5.json 2>gpurun_out/r2d/bench_cfg5.err; echo c5_exit=$?
timeout 900 python bench.py --config 4 --no-cpu --no-solve --steps 5 --warmup 3 > gpurun_out/r2d/bench_cfg4.json 2>gpurun_out/r2d/bench_cfg4.err; echo c4_exit=$?
timeout 900 python bench.py --config 3 --no-cpu --no-solve --steps 5 --warmup 3 > gpurun_out/r2d/bench_cfg3.json 2>gpurun_out/r2d/bench_cfg3.err; echo c3_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(hv_wc|eval)" -c 3 -o gpurun_out/r2d/k5 python bench.py --config 5 --no-cpu --no-solve --steps 1 --warmup 3 > gpurun_out/r2d/ncu5.log 2>&1; echo ncu5_exit=$?
for f in gpurun_out/r2d/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
rm -f gpurun_out/r2d/*.ncu-rep
