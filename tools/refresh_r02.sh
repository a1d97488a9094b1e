#!/bin/bash
# Round-2 evidence refresh wrapper: run final_refresh.sh, summarise the ncu captures ON the box (ncu -i),
# copy the summaries into gpurun_out/, and drop the big .ncu-rep files (gpurun merges <= 64 MiB back).
TAG=${1:-r02f}
NEXT=1 NEXT_ONLY="${NEXT_ONLY:-q16row q16frame frame adjoint closed_loop}" bash tools/final_refresh.sh $TAG
python tools/summarize_profile.py gpurun_out/$TAG $TAG > gpurun_out/$TAG/summarize.log 2>&1
python tools/summarize_next.py gpurun_out/$TAG-next $TAG >> gpurun_out/$TAG/summarize.log 2>&1
python tools/tabulate_bench.py gpurun_out/$TAG > gpurun_out/$TAG/bench_table.md 2>&1
mkdir -p gpurun_out/$TAG/profiles && cp profiles/${TAG}_* profiles/ncu_traffic.json gpurun_out/$TAG/profiles/ 2>/dev/null
du -sh gpurun_out/$TAG/*.ncu-rep gpurun_out/$TAG-next/*/*.ncu-rep > gpurun_out/$TAG/rep_sizes.txt 2>&1
find gpurun_out -name "*.ncu-rep" -size +8M -delete
du -sh gpurun_out >> gpurun_out/$TAG/rep_sizes.txt
