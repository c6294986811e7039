for z in 0 1 0 1; do SWB_ZALIGN=$z TAG=zalign$z timeout 300 python scripts/probe_k1perf.py 256:4 256:8 256:12 256:16 512:8 512:16; done
