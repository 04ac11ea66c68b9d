set -x
mkdir -p gpurun_out/r2o
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2o/pytest_all.log 2>&1; echo all_exit=$?; tail -3 gpurun_out/r2o/pytest_all.log
timeout 600 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "2,3" --steps 3 > gpurun_out/r2o/bench5.json 2>gpurun_out/r2o/bench5.err; echo b5_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/r2o/bench4.json 2>gpurun_out/r2o/bench4.err; echo b4_exit=$?
