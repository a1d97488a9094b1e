#!/bin/bash
# ncu --set full of one launch of the C4 kernel for the given M values (after a clean plain run).
TAG=${1:-prof}; MS=${2:-16}
OUT=gpurun_out/$TAG; mkdir -p $OUT
CMD="python bench.py --M $MS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
N=$(python -c "print(len('$MS'.split(',')))")
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_measure -s $((3*N)) -c $N -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu_full.log
tail -2 $OUT/ncu_full.log
