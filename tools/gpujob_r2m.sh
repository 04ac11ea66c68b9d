# Round-2 evidence: full default bench line, reference arm, launch list of the bench command, cfg4 line
set -x
mkdir -p gpurun_out/r2m
timeout 1200 python bench.py > gpurun_out/r2m/bench.json 2> gpurun_out/r2m/bench.err; echo bench_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --secondary "" --steps 5 > gpurun_out/r2m/bench_cfg4.json 2> gpurun_out/r2m/bench_cfg4.err; echo c4_exit=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2m/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-solve --e2e-steps 0 --secondary "" > gpurun_out/r2m/ncu_launch.log 2>&1; echo launch_exit=$?
