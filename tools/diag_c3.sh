#!/bin/bash
# C3 / per-config diagnostics: plan scan, CTA-0 timeline, ncu full captures of C2 / C3 / C5 (DRAM traffic
# per config).  usage: tools/diag_c3.sh [tag]   -> gpurun_out/<tag>/
TAG=${1:-diag}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "bench_candidate" > $OUT/pytest_cand.log 2>&1; echo "rc=$?" >> $OUT/pytest_cand.log
timeout 300 python tools/plan_scan.py C3 64 25 > $OUT/plan_scan_C3.log 2>&1
timeout 300 python tools/trace_timeline.py C3 64 > $OUT/trace_C3.log 2>&1
for wl in C3 C2 C5; do
  M=$(python -c "import synth; print(synth.CONFIGS['$wl'].M)")
  timeout 120 python tools/run_one.py $wl $M 3 > $OUT/plain_$wl.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cs_measure -s 2 -c 1 -o $OUT/prof_$wl python tools/run_one.py $wl $M 3 > $OUT/ncu_$wl.log 2>&1
  echo "ncu $wl rc=$?" >> $OUT/ncu_$wl.log
done
