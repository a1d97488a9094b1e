#!/bin/bash
for v in 0 1 2; do
  L=paper_1311_1419_b200/_lib/libcsenc_conv$v.so
  echo "variant $v: $(CSENC_LIB=$L python tools/gpu_debug.py | grep -c 'ok=True')/7 parity"
  CSENC_LIB=$L python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('  C4', round(d['value']), round(d['roofline']['frac'],3), {k:(round(v['gpix_s']),round(v['frac_of_peak'],3)) for k,v in d['per_M'].items()})"
  CSENC_LIB=$L python bench.py --workload C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('  C5', round(d['value']), round(d['roofline']['frac'],3))"
done
