set -x
mkdir -p gpurun_out/r2n
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "graph or dense_rho or pcg or eval_post" > gpurun_out/r2n/pytest_graph.log 2>&1; echo g_exit=$?; tail -3 gpurun_out/r2n/pytest_graph.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2n/pytest_all.log 2>&1; echo all_exit=$?; tail -3 gpurun_out/r2n/pytest_all.log
timeout 600 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2n/bench5.json 2>gpurun_out/r2n/bench5.err; echo b5_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2n/bench4.json 2>gpurun_out/r2n/bench4.err; echo b4_exit=$?
