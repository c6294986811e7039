#!/bin/bash
# Pencil-warp placement / split-point A/B at SO 16: default build against
# variants built with `python paper_1912_00695_b200/build.py --variant NAME -D...`.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in "" ${VARIANTS:-pw4 pw4k4 pw4k3 k4}; do
    if [ -n "$lib" ]; then
        export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so
    else
        unset SWB_LIB
    fi
    timeout 300 python scripts/probe_k1perf.py 256:16 512:16 ${EXTRA_CASES}
done
