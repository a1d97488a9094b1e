#!/bin/bash
# f2 ring-depth sweep (frames slots x A slots x residual buffers): TFLOP/s and fraction of the dense peak
for cfg in "" "CSENC_FRAME_ASLOTS=4" "CSENC_FRAME_ASLOTS=4 CSENC_FRAME_FSLOTS=4" "CSENC_FRAME_ASLOTS=3 CSENC_FRAME_FSLOTS=4" "CSENC_FRAME_ASLOTS=5" "CSENC_FRAME_ASLOTS=4 CSENC_FRAME_BBUFS=3" ""; do
  env $cfg timeout 300 python bench.py --op frame --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg', round(r['achieved'],1), round(r['frac'],3))" || echo "$cfg FAILED"
done
