#!/bin/bash
# sweep planner knobs for the C4 bench: each line = env setting -> per-M Gpix/s and HBM fraction
run() {
  env "$@" python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --M ${MS:-16,32} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), v['plan']['chunk_rows'], v['plan']['stages']) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$* FAILED"
}
for cfg in "CSENC_CHUNK_ROWS=16" "CSENC_CHUNK_ROWS=16 CSENC_STAGES=3" "CSENC_CHUNK_ROWS=16 CSENC_STAGES=2" "CSENC_CHUNK_ROWS=8" "CSENC_CHUNK_ROWS=16 CSENC_KEY_RESIDENT=0" "CSENC_TILE_ROWS=2 CSENC_CHUNK_ROWS=8"; do
  MS=16,32,64,128 run $cfg
done
