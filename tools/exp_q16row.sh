#!/bin/bash
# q16row A/B (libcsenc_old.so vs libcsenc.so) + the q16 / key-chunk / checks tests
OUT=gpurun_out/${1:-q16x}; mkdir -p $OUT; rm -f $OUT/ab.log
L=paper_1311_1419_b200/_lib
timeout 900 python -m pytest tests/test_gpu_q16.py tests/test_gpu_key_chunk.py tests/test_gpu_pdl.py tests/test_gpu_graph.py tests/test_gpu_checks.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
python bench.py --output q16row --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json > /dev/null 2>&1
for lib in libcsenc_old.so libcsenc.so libcsenc_old.so libcsenc.so; do
CSENC_LIB=$L/$lib python bench.py --output q16row --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', round(d['value'], 1), round(d['roofline']['frac'], 3), {k: round(v['ms_mean']*1e3,1) for k, v in d.get('per_M', {}).items()}, d['parity']['ok'])" >> $OUT/ab.log
done
