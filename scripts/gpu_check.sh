#!/bin/bash
# Standard GPU iteration: tests + perf of both kernel variants.
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} 2>&1 | tail -12
if [ -n "$SQ" ]; then SWB_KERNEL=sq timeout 200 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} 2>&1 | tail -12; fi
