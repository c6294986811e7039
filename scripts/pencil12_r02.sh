#!/bin/bash
# SO 12 y-pencil variant (28-row tile, 16 warps, pencil at warp 4) against the 15-warp default:
# (Needs the SO 12 pencil variant and the SWB_PENCIL_K6 / SWB_PENCIL_NSUB6 switches, which were measured and
# reverted; kept as the record of how profiles/pencil12_r02.txt was produced.)
# accuracy vs the bit-exact kernel and throughput (probe_pencil.py n:so:T1:YW:UNR), per build.
cd "$(dirname "$0")/.."
for lib in "" ${VARIANTS:-k6_3 k6_5 nsub1}; do
    if [ -n "$lib" ]; then
        export SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_$lib.so
    else
        unset SWB_LIB
    fi
    echo "== ${lib:-libswb.so}"
    timeout 300 python scripts/probe_pencil.py 256:12:28:0:4 256:12:28:1:2 256:12:28:1:4 512:12:28:1:2 512:12:28:0:4
done
