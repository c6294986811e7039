#!/bin/bash
mkdir -p gpurun_out
for lib in paper_1912_00695_b200/_lib/libswb.so paper_1912_00695_b200/_lib/variants/libswb_combine1.so paper_1912_00695_b200/_lib/variants/libswb_combine2.so; do
  SWB_LIB=$lib timeout 600 python scripts/probe_combine.py
done 2>&1 | tee gpurun_out/combine.log
for so in 8 16; do SWB_TRACE=1 timeout 120 python scripts/trace_launch.py $so 256; done 2>&1 | tee gpurun_out/trace.log
bash scripts/ncu_steady.sh 2>&1 | tail -8
