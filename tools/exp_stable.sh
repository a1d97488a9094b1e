#!/bin/bash
OUT=gpurun_out/stable; mkdir -p $OUT; rm -f $OUT/ab.log
timeout 900 python -m pytest tests/test_gpu_pdl.py tests/test_gpu_graph.py tests/test_gpu_q16.py tests/test_gpu_keys.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for W in C4 C3 C5; do
for S in 0 1 0 1; do
BENCH_STABLE_INPUTS=$S python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --workload $W 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$W stable=$S', round(d['value'], 1), round(d['ms_per_step']*1e3,1), round(d['roofline']['frac'], 3), d['parity']['ok'])" >> $OUT/ab.log
done; done
