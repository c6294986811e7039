#!/bin/bash
# A/B of the tile-height plan: makespan x T1^0.25 (default) vs row efficiency only (SWB_TPLAN=rows)
mkdir -p gpurun_out
for i in 1 2; do
for v in default rows; do
  SWB_TPLAN=$v TAG="plan_$v" timeout 600 python scripts/probe_k1perf.py 256:4 256:8 256:12 256:14 256:16 384:8 384:16 512:12 512:16 320:16 448:16
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q 2>&1 | tail -3
