#!/bin/bash
# A/B of programmatic dependent launch (CSENC_PDL=0 build vs the default) on one box
OUT=gpurun_out/pdl; mkdir -p $OUT
L=paper_1311_1419_b200/_lib
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_q16.py -m gpu -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for W in C2 C3 C4 C5; do
  echo "== $W" >> $OUT/ab.log
  bash tools/ab.sh $L/libcsenc_nopdl.so $L/libcsenc.so --workload $W >> $OUT/ab.log 2>&1
done
echo "== q16frame" >> $OUT/ab.log
bash tools/ab.sh $L/libcsenc_nopdl.so $L/libcsenc.so --output q16frame >> $OUT/ab.log 2>&1
