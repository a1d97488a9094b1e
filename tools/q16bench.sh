set -e
mkdir -p gpurun_out
TF=gpurun_out/tune_c4.json
for o in f32 q16row q16frame; do
  python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --tune-file $TF --output $o > gpurun_out/q16_$o.json
  python -c "import json; d=json.load(open('gpurun_out/q16_$o.json')); print('$o', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), {k:(round(v['gpix_s']),round(v['frac_of_peak'],3)) for k,v in d['per_M'].items()}, d['clocks']['sm_mhz'])"
done
