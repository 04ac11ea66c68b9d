# quick suite + ncu source capture of one dense kernel class at config 5
# usage: bash tools/gpujob_ncu1.sh TAG KERNEL_REGEX [SKIP] [COUNT]
set -x
T=${1:-q}; K=${2:-k_eval}; SKIP=${3:-2}; CNT=${4:-1}
bash tools/gpujob_quick.sh $T
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^($K)" --launch-skip $SKIP -c $CNT -o gpurun_out/$T/ncu python bench.py --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 1 --warmup 3 > gpurun_out/$T/ncu.log 2>&1; echo ncu_exit=$?
ncu -i gpurun_out/$T/ncu.ncu-rep --page raw --csv > gpurun_out/$T/ncu_raw.csv 2>/dev/null
ncu -i gpurun_out/$T/ncu.ncu-rep --page source --csv --print-source sass > gpurun_out/$T/ncu_sass.csv 2>/dev/null
rm -f gpurun_out/$T/ncu.ncu-rep
