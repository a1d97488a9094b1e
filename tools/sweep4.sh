#!/bin/bash
run() {
  env "$@" python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline --M ${MS:-16,32,128} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), round(240*1920*1080/v['ms_mean']/1e6)) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$* FAILED"
}
run CSENC_DBG_FLAGS=0
run CSENC_DBG_FLAGS=8
run CSENC_DBG_FLAGS=10
run CSENC_DBG_FLAGS=2
