set -e
mkdir -p gpurun_out
python bench.py --op closed_loop --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --tune-file gpurun_out/tune_c4.json > gpurun_out/cl_C4.json
python -c "import json; d=json.load(open('gpurun_out/cl_C4.json')); print('closed_loop C4', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), 'key ms', d['config']['key_codec_ms'], {k:(round(v['gpix_s']),round(v['frac_of_peak'],3)) for k,v in d['per_M'].items()})"
python bench.py --op encode --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --tune-file gpurun_out/tune_c4.json > gpurun_out/ol_C4.json
python -c "import json; d=json.load(open('gpurun_out/ol_C4.json')); print('open_loop C4', round(d['value'],1), 'frac', round(d['roofline']['frac'],3))"
