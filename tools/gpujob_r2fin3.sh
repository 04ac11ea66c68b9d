# Closing set, second pass (after the always-dense policy, the overlay rule, the dense-format roofline
# bytes and the warmed-up solve timing): whole GPU suite, default bench, reference arm, configs 4 and 3,
# launch list, and the config-5 hess_apply capture on a launch inside the CG (skip 20).
set -x
T=${1:-r2fin3}
mkdir -p gpurun_out/$T
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_all.log 2>&1; echo all_exit=$?; tail -5 gpurun_out/$T/pytest_all.log
timeout 1200 python bench.py > gpurun_out/$T/bench_full.json 2>gpurun_out/$T/bench_full.err; echo full_exit=$?
timeout 900 python bench.py --impl reference > gpurun_out/$T/bench_ref.json 2>gpurun_out/$T/bench_ref.err; echo ref_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench_cfg4.json 2>gpurun_out/$T/bench_cfg4.err; echo c4_exit=$?
timeout 600 python bench.py --config 3 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench_cfg3.json 2>gpurun_out/$T/bench_cfg3.err; echo c3_exit=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/$T/launches_cfg5_steps2.csv python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/$T/ncu_launch.log 2>&1; echo launch_exit=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_hv_wcd\$" --launch-skip 20 -c 1 -o gpurun_out/$T/full_c5_k_hv_wcd python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 1 --warmup 3 > gpurun_out/$T/full_c5_k_hv_wcd.log 2>&1; echo hv_exit=$?
ncu -i gpurun_out/$T/full_c5_k_hv_wcd.ncu-rep --page raw --csv > gpurun_out/$T/full_c5_k_hv_wcd_raw.csv 2>/dev/null
rm -f gpurun_out/$T/full_c5_k_hv_wcd.ncu-rep
python tools/bench_brief.py gpurun_out/$T/bench_full.json gpurun_out/$T/bench_cfg4.json gpurun_out/$T/bench_cfg3.json
