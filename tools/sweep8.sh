#!/bin/bash
run() {
  env "$@" python bench.py --workload $WL --steps 30 --warmup 4 --no-e2e --no-cpu-baseline ${MS:+--M $MS} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$WL', '$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), {x:v['plan'][x] for x in ('tile_block_rows','chunk_rows','stages','key_resident','a_bufs','d_bufs')}) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$WL $* FAILED"
}
for kr in 2 1; do WL=C5 run CSENC_KEY_RESIDENT=$kr; WL=C4 MS=16,32 run CSENC_KEY_RESIDENT=$kr; done
WL=C5 run CSENC_TILE_ROWS=2
WL=C5 run CSENC_TILE_ROWS=4
WL=C5 run CSENC_TILE_ROWS=6
