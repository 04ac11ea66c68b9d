# dense overlay at config 3: tests, then config-3 step + solve with and without the overlay
T=${1:-ov3}
mkdir -p gpurun_out/$T
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "overlay or dense_rho or config3" > gpurun_out/$T/pytest_ov.log 2>&1; echo ov_exit=$?; tail -15 gpurun_out/$T/pytest_ov.log
i=0
for E in "X=0" "OTB_HV_OVERLAY=0"; do
  i=$((i+1))
  env $E timeout 600 python bench.py --config 3 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/v$i.json 2>gpurun_out/$T/v$i.err || tail -3 gpurun_out/$T/v$i.err
  echo "== $E"; python tools/bench_brief.py gpurun_out/$T/v$i.json
  python -c "import json;d=json.loads(open('gpurun_out/$T/v$i.json').read().strip().splitlines()[-1]);g=d['details']['geometry'];print({k:g.get(k) for k in ('hv_mode','hv_grid','wc_nq','wc_win','wc_ncl','rho_dense')}, d['solve'])"
done
