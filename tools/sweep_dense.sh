# Dense-pass geometry sweep: consumer threads per CTA x CTAs per SM.
for cfg in 2 3; do
for combo in "512 1" "256 2" "128 4" "256 1"; do
  set -- $combo
  echo "== cfg$cfg NT=$1 CPS=$2"
  OTB_DENSE_NT=$1 OTB_DENSE_CTAS_PER_SM=$2 timeout 300 python bench.py --config $cfg --no-cpu --no-solve --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']['per_kernel']
print(round(d['value'],1), {k:round(v['us_per_launch'],1) for k,v in r.items()}, d['config']['geometry']['nt'], d['config']['geometry']['grid'])"
done; done
