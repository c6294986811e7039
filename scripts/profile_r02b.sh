#!/bin/bash
# Round-2b evidence on one B200: bench launch list + ncu --set full of K1 at SO 4-16 (profile_box.sh),
# steady-state DRAM ranges of the SO 16 kernels, summaries copied back through gpurun_out/.
bash scripts/profile_box.sh ${TAG:-r02b}
CFGS="16_256 16_512" bash scripts/ncu_steady.sh
python scripts/ncu_steady_summary.py ${TAG:-r02b} > gpurun_out/steady_summary.log 2>&1
cp profiles/ncu_summary.json profiles/ncu_steady_${TAG:-r02b}_*.csv gpurun_out/ 2>/dev/null
ls -la gpurun_out
