#!/bin/bash
OUT=gpurun_out/swz; mkdir -p $OUT; rm -f $OUT/ab.log
L=paper_1311_1419_b200/_lib
timeout 600 python -m pytest tests/test_gpu_key_chunk.py tests/test_gpu_phi_stream.py tests/test_gpu_parity.py tests/test_gpu_keys.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo "== C3 old / noswz / swz" >> $OUT/ab.log
for lib in libcsenc_old.so libcsenc_noswz.so libcsenc.so libcsenc_old.so libcsenc_noswz.so libcsenc.so; do
CSENC_LIB=$L/$lib python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload C3 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'], 1), round(d['roofline']['frac'], 3), {k: round(v['ms_mean']*1e3,1) for k, v in d.get('per_M', {}).items()})" >> $OUT/ab.log
done
python tools/plan_scan.py C3 64 6 > $OUT/plan_scan_C3.log 2>&1
BEST=$(grep -m1 "cand" $OUT/plan_scan_C3.log | awk '{print $4}'); echo "{\"C3:64\": $BEST}" > $OUT/tune.json
TUNE_FILE=$OUT/tune.json python tools/trace_timeline.py C3 64 > $OUT/trace_C3.log 2>&1
