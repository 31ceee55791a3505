python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in cfg2_nat_tiny_s1 cfg4_ade20k_128; do
 for lg in 0 1; do
  if [ $lg = 1 ]; then export NA2D_B1_LEGACY_ORDER=1; else unset NA2D_B1_LEGACY_ORDER; fi
  timeout 300 python bench.py --no-extras --steps 20 --warmup 5 --config $c > /tmp/o.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]); print('$c legacy=$lg', round(d['ms_per_step'],4), {k:round(v['avg_us'],1) for k,v in d['roofline']['kernels'].items()})"
 done
done
