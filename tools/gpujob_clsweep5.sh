# Dense-pass cluster-size sweep at config 5 (per-kernel us and it/s).
T=${1:-cl5}
mkdir -p gpurun_out/$T
for cl in 6 9 10 8; do
  env OTB_DENSE_CL=$cl timeout 600 python bench.py --config 5 --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/c5_cl$cl.json 2>gpurun_out/$T/c5_cl$cl.err
  echo "cl$cl exit=$?"
  python tools/bench_brief.py gpurun_out/$T/c5_cl$cl.json
done
