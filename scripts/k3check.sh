#!/bin/bash
# K3 development check: bitwise vs K1, repeatability, perf of both at 256^3.
for i in 1 2 3; do timeout 120 python scripts/k3_debug.py 12 2>&1 | grep -c "equal_K1=False"; done
timeout 600 python -m pytest tests/test_gpu_temporal.py -x -q 2>&1 | tail -4
TB=1 timeout 200 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} 256 200 2>&1 | tail -4
TB=2 timeout 200 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} 256 200 2>&1 | tail -4
