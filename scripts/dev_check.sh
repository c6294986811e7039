#!/bin/bash
# Development loop on one B200: GPU tests (optionally a -k filter) + K1 perf at 256^3.
timeout 600 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} 2>&1 | tail -3
timeout 300 python scripts/probe_perf.py factorised ${SOS:-4,8,12,16} 256 ${NT:-200} 2>&1 | tail -4
