for L in 1 2 3 5 7; do
  CSENC_LOOKBACK=$L python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --tune-file gpurun_out/tune_c4.json --output q16frame > gpurun_out/q16f_L$L.json
  python -c "import json; d=json.load(open('gpurun_out/q16f_L$L.json')); print('lag $L', round(d['value'],1), {k:round(v['gpix_s']) for k,v in d['per_M'].items()})"
done
