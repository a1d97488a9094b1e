#!/bin/bash
run() {
  env "$@" python bench.py --workload C4 --steps 30 --warmup 4 --no-e2e --no-cpu-baseline --M ${MS:-32,64,128} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), {x:v['plan'][x] for x in ('chunk_rows','stages','key_resident','a_bufs','d_bufs')}) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$* FAILED"
}
run X=0
run CSENC_KEY_RESIDENT=1
run CSENC_KEY_RESIDENT=1 CSENC_CHUNK_ROWS=8
run CSENC_KEY_RESIDENT=2 CSENC_STAGES=4
run CSENC_KEY_RESIDENT=2 CSENC_TMEM_BUFS=2,2
MS=16 run CSENC_KEY_RESIDENT=1
