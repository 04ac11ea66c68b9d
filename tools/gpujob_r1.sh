# Round-1 evidence: GPU tests, full bench line, ncu launch list and full
# capture of the step's kernels (each ncu run after the same command exited 0),
# CG phase trace, and the larger BASELINE configs.
set -x
mkdir -p gpurun_out/r1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r1/pytest_gpu.log 2>&1; echo pytest_exit=$?; tail -3 gpurun_out/r1/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r1/bench.json 2> gpurun_out/r1/bench.err; echo bench_exit=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/r1/bench_short.json 2>&1; echo short_exit=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r1/launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/r1/ncu_launch.log 2>&1; echo ncu_launch_exit=$?
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_(cg_fused|eval|sparsify|test_a|test_b|test_c)$" -c 7 -o gpurun_out/r1/full python bench.py --steps 1 --warmup 3 --no-solve --no-cpu > gpurun_out/r1/ncu_full.log 2>&1; echo ncu_full_exit=$?
OTB_CG_TRACE=1 timeout 300 python tools/hv_micro.py > gpurun_out/r1/cg_trace.txt 2>&1; echo trace_exit=$?
timeout 900 python bench.py --config 3 --no-cpu --no-solve --steps 10 --warmup 3 > gpurun_out/r1/bench_cfg3.json 2>/dev/null; echo c3_exit=$?
timeout 900 python bench.py --config 4 --no-cpu --no-solve --steps 5 --warmup 3 > gpurun_out/r1/bench_cfg4.json 2>/dev/null; echo c4_exit=$?
timeout 1200 python bench.py --config 5 --no-cpu --no-solve --steps 3 --warmup 3 > gpurun_out/r1/bench_cfg5.json 2>/dev/null; echo c5_exit=$?
