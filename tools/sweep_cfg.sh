#!/bin/bash
# Sweep forced K1 plans on one workload: each line = env setting -> Gpix/s, HBM fraction, plan.
# usage: WL=C3 tools/sweep_cfg.sh "CSENC_TILE_ROWS=3 CSENC_CHUNK_ROWS=8" "CSENC_TILE_ROWS=6 CSENC_CHUNK_ROWS=4" ...
WL=${WL:-C3}
for cfg in "$@"; do
  env $cfg timeout 120 python bench.py --workload $WL --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-autotune 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$WL $cfg', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), {q: v['plan'].get(q) for q in ('tile_block_rows','chunk_rows','key_resident','stages','a_bufs','d_bufs','phi_stream')}) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$WL $cfg FAILED"
done
