set -x
mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_rho or hess_apply or cluster_paths or step_pipeline or pcg" > gpurun_out/r2k/pytest.log 2>&1; echo t_exit=$?; tail -3 gpurun_out/r2k/pytest.log
timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2k/bench5.json 2>gpurun_out/r2k/bench5.err; echo b5_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_hv_wc" --launch-skip 50 -c 1 -o gpurun_out/r2k/hv5 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/r2k/ncu5.log 2>&1; echo ncuhv_exit=$?
for f in gpurun_out/r2k/*.ncu-rep; do ncu -i "$f" --page raw --csv > "${f%.ncu-rep}_raw.csv" 2>/dev/null; ncu -i "$f" --page source --csv --print-source sass > "${f%.ncu-rep}_sass.csv" 2>/dev/null; done
rm -f gpurun_out/r2k/*.ncu-rep
