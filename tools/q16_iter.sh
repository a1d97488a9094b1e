#!/bin/bash
# f1 per-frame (q16frame) iteration: build, the q16 / api / key-chunk / checks GPU tests, bench lines.
TAG=${1:-q16}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_q16.py tests/test_gpu_api.py tests/test_gpu_key_chunk.py tests/test_gpu_checks.py -q -x > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
tail -4 $OUT/pytest.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --output q16frame > $OUT/bench_q16frame.json 2> $OUT/bench_q16frame.err
python - <<PY
import json
d = json.loads(open("$OUT/bench_q16frame.json").read().strip().splitlines()[-1])
print("q16frame", round(d["value"]), round(d["roofline"]["frac"], 3), d.get("parity", {}).get("ok"), (d.get("e2e") or {}).get("value"))
for m, v in d["per_M"].items(): print(" M", m, round(v["ms_mean"] * 1e3, 1), "us", round(v["frac_of_peak"], 3))
PY
