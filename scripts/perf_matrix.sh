#!/bin/bash
# perf of kernel variants: each line ENV settings then probe output
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 200 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} ${N:-256} ${NT:-50} 2>&1 | tail -4
done
