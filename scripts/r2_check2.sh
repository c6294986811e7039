#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model_fields.py tests/test_gpu_dropin.py tests/test_gpu_fullsize.py tests/test_gpu_multidevice.py -x -q > gpurun_out/t2.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t2.log
for i in 1 2; do SWB_DROPIN_PROFILE=1 DROPIN_REPS=2 integration/_build/dropin_run aggressive 256 256 256 8 1000 0 - ; done 2>&1 | tail -16
SWB_DROPIN_PROFILE=1 integration/_build/dropin_run aggressive 256 256 256 8 1000 0.00002 - 2>&1 | tail -8
timeout 900 python scripts/probe_longrun_forms.py 128 4 8 16 > gpurun_out/longrun.log 2>&1; cat gpurun_out/longrun.log
