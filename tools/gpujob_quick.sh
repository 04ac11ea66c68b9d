# quick check after a kernel change: whole gpu suite, config-5 and config-4 step benches
# usage: bash tools/gpujob_quick.sh TAG
set -x
T=${1:-q}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_all.log 2>&1; echo all_exit=$?; tail -15 gpurun_out/$T/pytest_all.log
timeout 600 python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench5.json 2>gpurun_out/$T/bench5.err; echo b5_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench4.json 2>gpurun_out/$T/bench4.err; echo b4_exit=$?
python tools/bench_brief.py gpurun_out/$T/bench5.json gpurun_out/$T/bench4.json
