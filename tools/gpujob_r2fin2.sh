# Round-2 closing measurement set (command lines of profiles/r2/*_fin2*): whole GPU suite, default
# bench (config 5 + CPU reference sample + e2e + solve + configs 2-3), the reference arm, config 4
# and 3 step lines, the ncu launch list of a 2-step config-5 bench, and one ncu --set full capture
# per top kernel at config 5 plus hess_apply/eval at configs 4 and 3 (each only after the same
# command exited 0 without ncu).
set -x
T=${1:-r2fin2}
mkdir -p gpurun_out/$T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/$T/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/$T/pytest_all.log 2>&1; echo all_exit=$?; tail -5 gpurun_out/$T/pytest_all.log
timeout 1200 python bench.py > gpurun_out/$T/bench_full.json 2>gpurun_out/$T/bench_full.err; echo full_exit=$?
timeout 900 python bench.py --impl reference > gpurun_out/$T/bench_ref.json 2>gpurun_out/$T/bench_ref.err; echo ref_exit=$?
timeout 600 python bench.py --config 4 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench_cfg4.json 2>gpurun_out/$T/bench_cfg4.err; echo c4_exit=$?
timeout 600 python bench.py --config 3 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/bench_cfg3.json 2>gpurun_out/$T/bench_cfg3.err; echo c3_exit=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/$T/launches_cfg5_steps2.csv python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 2 > gpurun_out/$T/ncu_launch.log 2>&1; echo launch_exit=$?
cap() {  # cap CONFIG KERNEL SKIP
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$2\$" --launch-skip $3 -c 1 -o gpurun_out/$T/full_c$1_$2 python bench.py --config $1 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 1 --warmup 3 > gpurun_out/$T/full_c$1_$2.log 2>&1; echo c$1_$2_exit=$?
  ncu -i gpurun_out/$T/full_c$1_$2.ncu-rep --page raw --csv > gpurun_out/$T/full_c$1_$2_raw.csv 2>/dev/null
  rm -f gpurun_out/$T/full_c$1_$2.ncu-rep
}
for K in "k_hv_wcd:40" "k_eval:2" "k_test_c:1" "k_test_a:1" "k_sparsify_dense:1" "k_test_b:1"; do cap 5 ${K%%:*} ${K##*:}; done
cap 4 k_hv_wcd 40
cap 4 k_eval 2
cap 3 k_hv_wcd 40
python tools/bench_brief.py gpurun_out/$T/bench_full.json gpurun_out/$T/bench_cfg4.json gpurun_out/$T/bench_cfg3.json
