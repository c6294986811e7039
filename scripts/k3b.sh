timeout 300 python -m pytest tests/test_gpu_temporal.py -x -q 2>&1 | tail -2
TB=2 timeout 200 python scripts/probe_perf.py factorised 4,8,12,16 256 200 2>&1 | tail -4
python scripts/trace_k3.py 4 2>&1 | tail -3
TB=1 timeout 200 python scripts/probe_perf.py factorised 8,16 512 50 2>&1 | tail -2
TB=2 timeout 200 python scripts/probe_perf.py factorised 8,16 512 50 2>&1 | tail -2
