# Session-3 check after the container rebuild: GPU suite, smoke, default bench, configs 4 and 3.
T=${1:-r2s3a}
mkdir -p gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$T/gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/$T/pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/$T/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$T/smoke.log 2>&1; echo smoke_exit=$?
timeout 1200 python bench.py --no-cpu > gpurun_out/$T/bench_full.json 2>gpurun_out/$T/bench_full.err; echo full_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/bench_cfg4.json 2>gpurun_out/$T/bench_cfg4.err; echo c4_exit=$?
timeout 600 python bench.py --config 3 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench_cfg3.json 2>gpurun_out/$T/bench_cfg3.err; echo c3_exit=$?
python tools/bench_brief.py gpurun_out/$T/bench_full.json gpurun_out/$T/bench_cfg4.json gpurun_out/$T/bench_cfg3.json
