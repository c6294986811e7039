#!/bin/bash
# Round-2e evidence (aligned z tiles, H < 8): bench launch list + ncu --set full of K1 at SO 4-16
# (profile_box.sh), steady-state DRAM ranges of the SO 4-12 kernels, summaries back through gpurun_out/.
TAG=${TAG:-r02e}
bash scripts/profile_box.sh $TAG
CFGS="4_256 8_256 12_256 8_512 8_512_damp" bash scripts/ncu_steady.sh
python scripts/ncu_steady_summary.py $TAG > gpurun_out/steady_summary.log 2>&1
cp profiles/ncu_summary.json profiles/ncu_steady_${TAG}_*.csv gpurun_out/ 2>/dev/null
ls -la gpurun_out
