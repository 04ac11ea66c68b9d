# dense P_rho window-cluster hess_apply; suite + cfg4/5 bench + ncu
set -x
mkdir -p gpurun_out/r2e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_rho or hess_apply or cluster_paths or step_pipeline" > gpurun_out/r2e/pytest_dense.log 2>&1; echo dense_exit=$?; tail -5 gpurun_out/r2e/pytest_dense.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2e/pytest_all.log 2>&1; echo all_exit=$?; tail -5 gpurun_out/r2e/pytest_all.log
timeout 900 python bench.py --config 5 --no-cpu --no-solve --steps 3 --warmup 3 > gpurun_out/r2e/bench_cfg5.json 2>gpurun_out/r2e/bench_cfg5.err; echo c5_exit=$?
timeout 900 python bench.py --config 4 --no-cpu --no-solve --steps 5 --warmup 3 > gpurun_out/r2e/bench_cfg4.json 2>gpurun_out/r2e/bench_cfg4.err; echo c4_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(hv_wc|sparsify)" -c 4 -o gpurun_out/r2e/k5 python bench.py --config 5 --no-cpu --no-solve --steps 1 --warmup 3 > gpurun_out/r2e/ncu5.log 2>&1; echo ncu5_exit=$?
for f in gpurun_out/r2e/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
rm -f gpurun_out/r2e/*.ncu-rep
