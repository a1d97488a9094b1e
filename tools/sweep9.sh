#!/bin/bash
run() {
  env "$@" python bench.py --workload C5 --steps 30 --warmup 4 --no-e2e --no-cpu-baseline 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C5', '$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), {x:v['plan'][x] for x in ('tile_block_rows','chunk_rows','stages','key_resident','a_bufs','d_bufs')}) for k,v in d['per_M'].items()})" 2>/dev/null || echo "C5 $* FAILED"
}
for i in 1 2 3; do run X=$i; done
for i in 1 2; do run CSENC_TMEM_BUFS=2,2; done
for i in 1 2; do run CSENC_KEY_RESIDENT=1 CSENC_TMEM_BUFS=2,2; done
