#!/bin/bash
# quick GPU iteration: parity smoke over all configs, pipeline trace, short bench summary
timeout 300 python tools/gpu_debug.py 2>&1 | grep -E "ok=|elapsed|Error|error" | cut -c1-120
python tools/trace_timeline.py C4 ${1:-16,128} 2>&1 | grep -v "^ *[0-9]"
python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', round(d['value'],1), 'frac', round(d['roofline']['frac'],3), {k:(round(v['gpix_s']),round(v['frac_of_peak'],3)) for k,v in d['per_M'].items()}, d['clocks'])"
