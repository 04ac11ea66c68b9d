# Round 2: new window-cluster hess_apply; whole GPU suite; cfg4/cfg5 bench; ncu of k_hv_wc
set -x
mkdir -p gpurun_out/r2c
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2c/pytest_all.log 2>&1; echo all_exit=$?; tail -15 gpurun_out/r2c/pytest_all.log
timeout 900 python bench.py --config 5 --no-cpu --no-solve --steps 3 --warmup 3 > gpurun_out/r2c/bench_cfg5.json 2>gpurun_out/r2c/bench_cfg5.err; echo c5_exit=$?
timeout 900 python bench.py --config 4 --no-cpu --no-solve --steps 5 --warmup 3 > gpurun_out/r2c/bench_cfg4.json 2>gpurun_out/r2c/bench_cfg4.err; echo c4_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_hv_wc" -c 2 -o gpurun_out/r2c/hv5 python bench.py --config 5 --no-cpu --no-solve --steps 1 --warmup 3 > gpurun_out/r2c/ncu5.log 2>&1; echo ncu5_exit=$?
for f in gpurun_out/r2c/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; done
tot=$(du -sm gpurun_out | cut -f1); if [ "$tot" -gt 60 ]; then rm -f gpurun_out/r2c/*.ncu-rep; fi
