#!/bin/bash
# load-only / no-store / no-convert ablations of one workload's step on a CSENC_DEBUG=1 CSENC_TUNING=1
# build (DESIGN.md sec.7 table).  usage: tools/dbg_ablation.sh [bench args, e.g. --workload C3]
L=paper_1311_1419_b200/_lib
[ -f $L/libcsenc_dbg.so ] || python -c "from paper_1311_1419_b200 import _build; _build.build(out='$L/libcsenc_dbg.so', defines=('CSENC_DEBUG=1', 'CSENC_TUNING=1'))"
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --tune-file /tmp/t.json "$@" > /dev/null 2>&1
for e in "" "CSENC_DBG_FLAGS=8" "CSENC_DBG_LOAD_ONLY=1" "CSENC_DBG_FLAGS=2" "CSENC_DBG_FLAGS=10"; do
  env $e CSENC_LIB=$L/libcsenc_dbg.so python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --tune-file /tmp/t.json "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$e', {k:(round(v['ms_mean']*1e3,1), round(v['gpix_s'])) for k,v in d['per_M'].items()})"
done
