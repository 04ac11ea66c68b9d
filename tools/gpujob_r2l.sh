set -x
mkdir -p gpurun_out/r2l
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2l/pytest_all.log 2>&1; echo all_exit=$?; tail -5 gpurun_out/r2l/pytest_all.log
timeout 900 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "1,2,3" --steps 3 > gpurun_out/r2l/bench5.json 2>gpurun_out/r2l/bench5.err; echo b5_exit=$?
timeout 900 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/r2l/bench4.json 2>gpurun_out/r2l/bench4.err; echo b4_exit=$?
