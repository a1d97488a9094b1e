for L in paper_1311_1419_b200/_lib/libcsenc_head.so paper_1311_1419_b200/_lib/libcsenc.so paper_1311_1419_b200/_lib/libcsenc_head.so paper_1311_1419_b200/_lib/libcsenc.so; do
  CSENC_LIB=$L python bench.py --op frame --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/f2ab.json
  python -c "import json; d=json.load(open('gpurun_out/f2ab.json')); print('$L', round(d['roofline']['achieved']), round(d['roofline']['frac'],3))"
done
