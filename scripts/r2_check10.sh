#!/bin/bash
# Round-2 evidence: ncu launch list of the default bench command + one --set full capture of K1 per
# SO (summarised on the box), and the long-run FP32 error table (128^3, 10k steps).
mkdir -p gpurun_out
bash scripts/profile_box.sh r02 > gpurun_out/profile_box.log 2>&1; echo "profile rc=$?"
cat gpurun_out/ncu_summary_r02.log | head -20
timeout 1200 python scripts/probe_longrun_forms.py 128 4 8 12 16 > gpurun_out/longrun.log 2>&1; echo "longrun rc=$?"
cat gpurun_out/longrun.log
