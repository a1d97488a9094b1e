#!/bin/bash
run() {
  env "$@" python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --M ${MS:-16} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
for M,v in d['per_M'].items():
  ms=v['ms_mean']; print('$*', 'M',M,'ms=%.3f'%ms, 'input GB/s=%.0f'%(240*1920*1080/ms/1e6), 'gpix %.0f frac %.3f'%(v['gpix_s'],v['frac_of_peak']), 'plan', v['plan']['chunk_rows'], v['plan']['stages'], v['plan']['key_resident'])" || echo "$* FAILED"
}
for sp in 0 16384 8192 4096 2048 1024; do run CSENC_DBG_LOAD_ONLY=1 CSENC_CHUNK_ROWS=8 CSENC_COPY_SPLIT=$sp; done
for sp in 4096 2048; do run CSENC_DBG_LOAD_ONLY=1 CSENC_CHUNK_ROWS=16 CSENC_COPY_SPLIT=$sp; done
MS=16,32,64,128 run CSENC_COPY_SPLIT=4096
MS=16,32,64,128 run CSENC_COPY_SPLIT=2048
