# Dense-pass cluster-size sweep at configs 5 and 4 (per-kernel us and it/s).
T=${1:-s3cl}
mkdir -p gpurun_out/$T
for cfg in 5 4; do
for cl in 0 4 6 8 9 10; do
  if [ $cl = 0 ]; then E=""; else E="OTB_DENSE_CL=$cl"; fi
  env $E timeout 600 python bench.py --config $cfg --no-cpu --no-solve --e2e-steps 0 --secondary "" --steps 3 > gpurun_out/$T/c${cfg}_cl$cl.json 2>gpurun_out/$T/c${cfg}_cl$cl.err
  echo "cfg$cfg cl$cl exit=$?"
  python tools/bench_brief.py gpurun_out/$T/c${cfg}_cl$cl.json
  python -c "import json;d=json.load(open('gpurun_out/$T/c${cfg}_cl$cl.json'));print(d['config'].get('geometry'))"
done; done
