#!/bin/bash
# Round-2f/2g evidence (r02g: final kernel with pencil variants at SO 8/12/16, P_y in the aux ring): ncu --set full of
# K1 at SO 4-16 + the bench launch list (profile_box.sh), steady-state DRAM of every 256^3 / 512^3 case.
TAG=${TAG:-r02f}
bash scripts/profile_box.sh $TAG
CFGS="4_256 8_256 12_256 16_256 8_512 8_512_damp 16_512" bash scripts/ncu_steady.sh
python scripts/ncu_steady_summary.py $TAG > gpurun_out/steady_summary.log 2>&1
cp profiles/ncu_summary.json profiles/ncu_steady_${TAG}_*.csv gpurun_out/ 2>/dev/null
ls -la gpurun_out
