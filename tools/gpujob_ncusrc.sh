# ncu --set full source-level captures (SASS stall samples) of named kernels at config 5
# usage: bash tools/gpujob_ncusrc.sh TAG "k_test_b:1 k_eval:2"
set -x
T=${1:-ncusrc}
mkdir -p gpurun_out/$T
for K in $2; do
  N=${K%%:*}; S=${K##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$N" --launch-skip $S -c 1 -o gpurun_out/$T/ncu_$N python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 1 --warmup 3 > gpurun_out/$T/ncu_$N.log 2>&1; echo ncu_${N}_exit=$?
  ncu -i gpurun_out/$T/ncu_$N.ncu-rep --page raw --csv > gpurun_out/$T/ncu_${N}_raw.csv 2>/dev/null
  ncu -i gpurun_out/$T/ncu_$N.ncu-rep --page source --csv --print-source sass > gpurun_out/$T/ncu_${N}_sass.csv 2>/dev/null
  rm -f gpurun_out/$T/ncu_$N.ncu-rep
done
