#!/bin/bash
# Round-end evidence refresh: smoke, GPU tests, the default bench line (headline, with e2e and the CPU
# baseline), the reference arm, one line per workload / op / output variant, and the ncu launch list +
# full capture of the headline step.  -> gpurun_out/<tag>/
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --tune-file $OUT/plans.json > $OUT/bench_C4.json 2> $OUT/bench_C4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
run () { local name=$1; shift; timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "$@" > $OUT/bench_$name.json 2> $OUT/bench_$name.err; }
run C1 --workload C1
run C2 --workload C2
run C3 --workload C3
run C5 --workload C5
run C4_q16row --output q16row
run C4_q16frame --output q16frame
run C4_adjoint --op adjoint
run C5_adjoint --op adjoint --workload C5
run C4_closed_loop --op closed_loop --tune-file $OUT/plans.json
run C4_gop_phis --gop-phis --tune-file $OUT/plans.json
run C5_gop_phis --gop-phis --workload C5
run f2_frame --op frame --steps 20
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cs_measure -s 12 -c 4 -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
echo "ncu rc=$?" >> $OUT/ncu_full.log
[ "${NEXT:-0}" = "1" ] && ONLY="${NEXT_ONLY:-q16row q16frame}" bash tools/prof_next.sh $TAG-next
