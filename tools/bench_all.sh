#!/bin/bash
# one bench line per workload (short) -> gpurun_out/<tag>/bench_<W>.json
TAG=${1:-all}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for w in C1 C2 C3 C4 C5; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-30} --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_$w.json 2> $OUT/bench_$w.err
  python -c "import json; d=json.load(open('$OUT/bench_$w.json')); print('$w', round(d['value'],1), 'Gpx/s frac', round(d['roofline']['frac'],3), {k:(round(v['gpix_s']),round(v['frac_of_peak'],3),round(v['ms_mean'],4)) for k,v in d['per_M'].items()})" || tail -3 $OUT/bench_$w.err
done
