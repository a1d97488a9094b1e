#!/bin/bash
# ncu evidence for the section-8 "next" rows: per op a plain run (must exit 0), the launch list
# (gpu__time_duration, --clock-control none) and one --set full capture of the op's main kernel.
# usage: tools/prof_next.sh [tag]      -> gpurun_out/<tag>/<op>/{bench.json,launches.csv,prof.ncu-rep}
TAG=${1:-r01next}
run_op () {  # name, kernel regex, skip, count, bench args...   (ONLY="a b" restricts to those ops)
  local name=$1 rx=$2 skip=$3 cnt=$4; shift 4
  if [ -n "$ONLY" ] && [[ " $ONLY " != *" $name "* ]]; then return; fi
  local OUT=gpurun_out/$TAG/$name
  mkdir -p $OUT
  local CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json $*"
  timeout 600 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $OUT/plans.json "$@" > $OUT/bench.json 2> $OUT/bench.err || { echo "$name bench failed"; return; }
  timeout 300 $CMD > $OUT/plain.log 2>&1 || { echo "$name plain failed"; return; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c $cnt -o $OUT/prof $CMD > $OUT/ncu_full.log 2>&1
  echo "$name done rc=$?"
}
run_op q16row cs_measure 12 4 --output q16row
run_op q16frame cs_measure 24 2 --output q16frame
run_op adjoint cs_adjoint 12 4 --op adjoint
run_op closed_loop key_codec 4 1 --op closed_loop
run_op frame frame_measure 3 1 --op frame
run_op adjoint_c5 cs_adjoint 3 1 --op adjoint --workload C5
