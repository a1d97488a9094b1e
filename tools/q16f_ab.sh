for fl in 0 48; do
  CSENC_LIB=paper_1311_1419_b200/_lib/libcsenc_dbg.so CSENC_DBG_FLAGS=$fl python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-autotune --output q16frame --M 16,128 > gpurun_out/q16f_$fl.json
  python -c "import json; d=json.load(open('gpurun_out/q16f_$fl.json')); print('dbg flags $fl', round(d['value'],1), {k:round(v['gpix_s']) for k,v in d['per_M'].items()})"
done
python -m pytest tests/test_gpu_q16.py -x -q 2>&1 | tail -1
bash tools/q16bench.sh
