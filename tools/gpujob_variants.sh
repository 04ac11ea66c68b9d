# Side-by-side library variants (_exp/<v>/libotb.so through OTB_LIB): config-5 and config-4 step benches
# usage: bash tools/gpujob_variants.sh TAG "v1 v2 ..." [configs]
T=${1:-var}
mkdir -p gpurun_out/$T
for v in $2; do
  for cfg in ${3:-5 4}; do
    OTB_LIB=$PWD/_exp/$v/libotb.so timeout 600 python bench.py --config $cfg --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/${v}_c$cfg.json 2>gpurun_out/$T/${v}_c$cfg.err || tail -3 gpurun_out/$T/${v}_c$cfg.err
    python tools/bench_brief.py gpurun_out/$T/${v}_c$cfg.json
  done
done
