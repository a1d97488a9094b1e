# A/B the key codec builds on the same box: closed-loop bench key_codec_ms per library
for L in paper_1311_1419_b200/_lib/libcsenc_kc3.so paper_1311_1419_b200/_lib/libcsenc_kc4.so paper_1311_1419_b200/_lib/libcsenc.so; do
  CSENC_LIB=$L python bench.py --op closed_loop --M 16 --steps 30 --warmup 3 --no-e2e --no-cpu-baseline --no-autotune > gpurun_out/kc.json
  python -c "import json; d=json.load(open('gpurun_out/kc.json')); print('$L', 'key ms', round(d['config']['key_codec_ms'],4))"
done
