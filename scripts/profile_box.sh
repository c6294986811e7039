#!/bin/bash
# Run the ncu evidence capture on the box and summarise it there (the .ncu-rep files of all
# captures exceed gpurun's 64 MiB return limit): keeps the text/JSON summaries, the launch
# list and the SO 8 / SO 16 K1 reports.
TAG=${1:-r01}
bash scripts/profile.sh > gpurun_out/profile.log 2>&1
python scripts/ncu_summary.py $TAG > gpurun_out/ncu_summary_$TAG.log 2>&1
cp profiles/ncu_summary.json profiles/ncu_k_tma_$TAG.txt gpurun_out/ 2>/dev/null
python scripts/launch_summary.py gpurun_out/launches.csv gpurun_out/launches_$TAG.txt "python bench.py (first 400 launches)" > /dev/null 2>&1
rm -f gpurun_out/tma_so4.ncu-rep gpurun_out/tma_so12.ncu-rep gpurun_out/tb_so*.ncu-rep
ls -la gpurun_out
