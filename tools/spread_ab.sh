for sp in 0 1; do
 for w in C3 C4 C5 C2; do
  CSENC_LANE_SPREAD=$sp python bench.py --workload $w --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sp.json
  python -c "import json; d=json.load(open('gpurun_out/sp.json')); print('spread $sp $w', round(d['value'],1), round(d['roofline']['frac'],3), {k:round(v['gpix_s']) for k,v in d['per_M'].items()})"
 done
done
