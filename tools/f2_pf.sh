for pf in 0 4 8 16; do
  CSENC_FRAME_PREFETCH=$pf python bench.py --op frame --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f2_pf$pf.json
  python -c "import json; d=json.load(open('gpurun_out/f2_pf$pf.json')); print('prefetch $pf', round(d['roofline']['achieved']), round(d['roofline']['frac'],3))"
done
