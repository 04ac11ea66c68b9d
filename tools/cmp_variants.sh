#!/bin/bash
# Compare library variants built into _exp/<v>/libotb.so (debug tool):
#   tools/cmp_variants.sh "a:OTB_DENSE_NT=384" "b:OTB_DENSE_NT=256" ...
# "base" runs the in-tree build.  Prints Newton it/s and per-kernel us.
cp paper_2603_07156_b200/libotb.so /tmp/libotb_base.so
for spec in base "$@"; do
  v=${spec%%:*}; envs=${spec#*:}; [ "$spec" = base ] && envs=""
  if [ "$v" = base ]; then cp /tmp/libotb_base.so paper_2603_07156_b200/libotb.so; else cp _exp/$v/libotb.so paper_2603_07156_b200/libotb.so; fi
  env $envs python bench.py --no-cpu --no-solve --steps 20 --warmup 3 --e2e-steps 0 ${BENCH_ARGS} > gpurun_out/cmp_$v.json 2>gpurun_out/cmp_$v.err
  python -c "import json,sys;d=json.load(open('gpurun_out/cmp_$v.json'));print('$spec', round(d['value'],1), {k:round(x['us_per_launch'],1) for k,x in d['roofline']['per_kernel'].items()})" || tail -3 gpurun_out/cmp_$v.err
done
cp /tmp/libotb_base.so paper_2603_07156_b200/libotb.so
