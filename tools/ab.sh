#!/bin/bash
# A/B the current library against paper_1311_1419_b200/_lib/libcsenc_old.so on the same box
for wl in C5 C4; do
 for L in paper_1311_1419_b200/_lib/libcsenc_old.so paper_1311_1419_b200/_lib/libcsenc.so; do
  CSENC_LIB=$L python bench.py --workload $wl --steps 30 --warmup 4 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$wl', '$(basename $L)', round(d['value']), round(d['roofline']['frac'],3), {k:round(v['gpix_s']) for k,v in d['per_M'].items()})"
 done
done
