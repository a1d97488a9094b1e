#!/bin/bash
# A/B two builds of the library on the SAME box (box-to-box spread is several percent):
#   tools/ab.sh LIB_A LIB_B [bench.py args...]     e.g. tools/ab.sh _lib/libcsenc_old.so _lib/libcsenc.so --op frame
# Runs A, B, A, B and prints value / roofline fraction / per-launch time of each run.
A=$1; B=$2; shift 2
for L in "$A" "$B" "$A" "$B"; do
  CSENC_LIB=$L python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$(basename $L)', round(d['value'], 1), round(d['roofline']['frac'], 3), d.get('per_launch_ms') or {k: round(v['gpix_s']) for k, v in d.get('per_M', {}).items()})"
done
