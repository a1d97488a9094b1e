#!/bin/bash
run() {
  env "$@" python bench.py --workload $WL --steps 20 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$WL', '$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), round(v['ms_mean'],4), {x:v['plan'][x] for x in ('tile_block_rows','folds','chunk_rows','stages','key_resident')}) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$WL $* FAILED"
}
WL=C3 run X=0
WL=C3 run CSENC_PREFETCH=8
WL=C3 run CSENC_TILE_ROWS=3 CSENC_CHUNK_ROWS=8
WL=C3 run CSENC_TILE_ROWS=3 CSENC_CHUNK_ROWS=8 CSENC_PREFETCH=6
WL=C3 run CSENC_TILE_ROWS=6 CSENC_CHUNK_ROWS=4
WL=C3 run CSENC_TILE_ROWS=6 CSENC_CHUNK_ROWS=4 CSENC_PREFETCH=8
WL=C3 run CSENC_TILE_ROWS=2 CSENC_CHUNK_ROWS=8 CSENC_KEY_RESIDENT=1
WL=C2 run X=0
WL=C2 run CSENC_TILE_ROWS=2
WL=C2 run CSENC_TILE_ROWS=1
WL=C2 run CSENC_PREFETCH=4
