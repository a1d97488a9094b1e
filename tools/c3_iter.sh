#!/bin/bash
# C3 iteration loop: KEY_CHUNK tests, plan scan, CTA-0 timeline of the best plan.  -> gpurun_out/<tag>/
TAG=${1:-c3}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_key_chunk.py tests/test_gpu_phi_stream.py tests/test_gpu_checks.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
timeout 300 python tools/plan_scan.py C3 64 ${TOP:-12} > $OUT/plan_scan_C3.log 2>&1
head -${TOP:-12} $OUT/plan_scan_C3.log | cut -c1-60
BEST=$(grep -m1 "cand" $OUT/plan_scan_C3.log | awk '{print $4}')
echo "{\"C3:64\": $BEST}" > $OUT/tune.json
TUNE_FILE=$OUT/tune.json timeout 300 python tools/trace_timeline.py C3 64 > $OUT/trace_C3.log 2>&1
head -14 $OUT/trace_C3.log
