#!/bin/bash
# u-ring depth of the pencil variants (SWB_SU selects; SWB_UNR=3 so the SO 12 / 16 variants match first).
# (Needs the measured-and-removed SU variants in SWB_TMA_VARIANTS; kept as the record of profiles/su_r02.txt.)
cd "$(dirname "$0")/.."
for pass in 1 2; do
  for su in 9 10 11; do SWB_UNR=3 SWB_SU=$su TAG="SO12 SU $su" timeout 300 python scripts/probe_k1perf.py 256:12 512:12; done
  for su in 12 13 14; do SWB_UNR=3 SWB_SU=$su TAG="SO16 SU $su" timeout 300 python scripts/probe_k1perf.py 256:16 512:16; done
  for su in 7 8 10; do SWB_SU=$su TAG="SO8 SU $su" timeout 300 python scripts/probe_k1perf.py 256:8 512:8; done
done
