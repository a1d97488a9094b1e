for nb in 2 3 4; do
  CSENC_FRAME_BBUFS=$nb python bench.py --op frame --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f2_nb$nb.json
  python -c "import json; d=json.load(open('gpurun_out/f2_nb$nb.json')); print('B bufs $nb', round(d['roofline']['achieved']), round(d['roofline']['frac'],3))"
done
