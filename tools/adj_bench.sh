set -e
mkdir -p gpurun_out
python bench.py --op adjoint --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/adj_C4.json
python -c "import json; d=json.load(open('gpurun_out/adj_C4.json')); print('adjoint C4', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), {k:(round(v['gpix_s']),round(v['frac_of_peak'],3), round(v['tflops_tf32'])) for k,v in d['per_M'].items()}, d['clocks']['sm_mhz'])"
python bench.py --op adjoint --workload C5 --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/adj_C5.json
python -c "import json; d=json.load(open('gpurun_out/adj_C5.json')); print('adjoint C5', round(d['value'],1), 'frac', round(d['roofline']['frac'],3))"
