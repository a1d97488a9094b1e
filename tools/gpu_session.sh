#!/bin/bash
# One gpurun session: GPU tests, bench, ncu launch list + one full capture of the kernel.
# usage: tools/gpu_session.sh [tag]
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 --tune-file $OUT/plans.json > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json"
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 $CMD > $OUT/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_measure -s 12 -c 4 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
  echo "ncu rc=$?" >> $OUT/ncu_full.log
fi
