#!/bin/bash
mkdir -p gpurun_out
V=paper_1912_00695_b200/_lib/variants
for lib in $V/libswb_lap1.so $V/libswb_lap2.so $V/libswb_lap2c2.so; do
  SWB_LIB=$lib timeout 600 python scripts/probe_combine.py
done 2>&1 | tee gpurun_out/lap.log
for mb in 0 64 100 200; do TAG="persist${mb}MB" SWB_L2_PERSIST=$mb timeout 300 python scripts/probe_k1perf.py; done 2>&1 | tee gpurun_out/l2.log
for mb in 0 200; do TAG="predel_persist${mb}MB" SWB_LIB=$V/libswb_predel.so SWB_L2_PERSIST=$mb timeout 300 python scripts/probe_k1perf.py 256:4 256:12; done 2>&1 | tee -a gpurun_out/l2.log
SWB_L2_PERSIST=200 timeout 600 ncu --cache-control none --clock-control none -k regex:k_tma -s 30 -c 12 --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv python scripts/ncu_steady.py 8 256 > gpurun_out/ncu_steady_persist_8_256.csv 2>&1
python - <<'PY'
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if False else None
PY
