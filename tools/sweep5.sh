#!/bin/bash
run() {
  env "$@" python bench.py --workload ${WL:-C4} --steps 20 --warmup 4 --no-e2e --no-cpu-baseline ${MS:+--M $MS} 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${WL:-C4}', '$*', {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), v['plan']['a_bufs'], v['plan']['d_bufs'], v['plan']['chunk_rows']) for k,v in d['per_M'].items()})" 2>/dev/null || echo "$* FAILED"
}
MS=16,32,64,128 run CSENC_TMEM_BUFS=2,2
MS=16,32,64,128 run X=1
MS=16,32 run CSENC_TMEM_BUFS=2,4
MS=16,32 run CSENC_TMEM_BUFS=3,3
MS=128 run CSENC_CHUNK_ROWS=8
WL=C5 run CSENC_TMEM_BUFS=2,2
WL=C5 run X=1
