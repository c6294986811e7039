#!/bin/bash
# compute-sanitizer pass over every kernel family + per-CTA traces of K1 at SO 8/16 (256^3)
mkdir -p gpurun_out
for so in 4 8 12 16; do timeout 120 python scripts/trace_launch.py $so 256; done 2>&1 | tee gpurun_out/trace.log
bash scripts/sanitize.sh 2>&1 | tee gpurun_out/sanitize_summary.txt
