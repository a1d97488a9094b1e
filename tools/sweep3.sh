#!/bin/bash
run() {
  env "$@" python bench.py --steps 20 --warmup 4 --no-e2e --no-cpu-baseline --M 16 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for M,v in d['per_M'].items():
  ms=v['ms_mean']; print('$*', 'ms=%.3f'%ms, 'input GB/s=%.0f'%(240*1920*1080/ms/1e6), 'plan', v['plan']['tile_block_rows'], v['plan']['chunk_rows'], v['plan']['stages'], v['plan']['key_resident'], v['plan']['prefetch_items'])" || echo "$* FAILED"
}
L="CSENC_DBG_LOAD_ONLY=1"
run $L CSENC_CHUNK_ROWS=8
run $L CSENC_CHUNK_ROWS=8 CSENC_PREFETCH=0
run $L CSENC_CHUNK_ROWS=16 CSENC_PREFETCH=0
run $L CSENC_CHUNK_ROWS=16 CSENC_PREFETCH=0 CSENC_TILE_ROWS=2
run $L CSENC_CHUNK_ROWS=8 CSENC_PREFETCH=0 CSENC_TILE_ROWS=2
run $L CSENC_CHUNK_ROWS=8 CSENC_PREFETCH=0 CSENC_TILE_ROWS=4
