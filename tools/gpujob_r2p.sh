# re-entry check: whole gpu suite, default bench (config 5), config 4 line
set -x
mkdir -p gpurun_out/r2p
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2p/pytest_all.log 2>&1; echo all_exit=$?; tail -3 gpurun_out/r2p/pytest_all.log
timeout 900 python bench.py > gpurun_out/r2p/bench_full.json 2>gpurun_out/r2p/bench_full.err; echo b5_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2p/bench4.json 2>gpurun_out/r2p/bench4.err; echo b4_exit=$?
