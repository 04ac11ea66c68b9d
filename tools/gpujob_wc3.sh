# config 3 (n = 10000): group kernel vs window clusters (dense / bitmap P_rho)
T=${1:-wc3}
mkdir -p gpurun_out/$T
i=0
for E in "X=0" "OTB_HV_WC=1" "OTB_HV_WC=1 OTB_HV_DENSE=0" "OTB_HV_WC=1 OTB_HV_NQ=5" "OTB_HV_WC=1 OTB_HV_NQ=4" "OTB_HV_WC=1 OTB_HV_NQ=2"; do
  i=$((i+1))
  env $E timeout 600 python bench.py --config 3 --no-cpu --e2e-steps 0 --secondary "" --steps 5 > gpurun_out/$T/v$i.json 2>gpurun_out/$T/v$i.err || tail -3 gpurun_out/$T/v$i.err
  echo "== $E"; python tools/bench_brief.py gpurun_out/$T/v$i.json
  python -c "import json;d=json.loads(open('gpurun_out/$T/v$i.json').read().strip().splitlines()[-1]);g=d['details']['geometry'];print({k:g[k] for k in ('hv_mode','hv_grid','hv_groups','hv_smem_bytes')}, d['solve']['time_s'], d['solve']['cg'], d['clocks'])"
done
