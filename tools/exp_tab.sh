#!/bin/bash
OUT=gpurun_out/tab; mkdir -p $OUT
L=paper_1311_1419_b200/_lib
python tools/plan_scan.py C3 64 14 > $OUT/plan_scan_C3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_key_chunk.py tests/test_gpu_phi_stream.py tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for W in C3 C4 C2 C5; do
  echo "== $W" >> $OUT/ab.log
  bash tools/ab.sh $L/libcsenc_old.so $L/libcsenc.so --workload $W >> $OUT/ab.log 2>&1
done
