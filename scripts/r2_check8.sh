#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_opsgen_b200.py -x -q > gpurun_out/opsgen.log 2>&1; echo "opsgen rc=$?"; tail -3 gpurun_out/opsgen.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool initcheck --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py slabs_ordered > gpurun_out/sanitize_initcheck_slabs_ordered.log 2>&1
echo "initcheck slabs_ordered rc=$? $(grep -h 'ERROR SUMMARY' gpurun_out/sanitize_initcheck_slabs_ordered.log | tail -1)"
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_hold$i.json 2> gpurun_out/bench_hold$i.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_hold$i.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], {k:v['gpts'] for k,v in d['sweep'].items()}, d['damped']['gpts'])"; done
