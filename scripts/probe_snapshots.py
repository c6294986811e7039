"""Overlap of snapshot drains with stepping: 256^3 SO 8, nt steps, a snapshot every `every`
steps into pinned host buffers, against the same steps without snapshots (development)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

n, so = 256, 8
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
every = int(sys.argv[2]) if len(sys.argv) > 2 else 50
prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=nt + 20))
bufs = [torch.empty((n, n, n), dtype=torch.float32, pin_memory=True).numpy() for _ in range(nt // every)]
op = P.Operator(prob)
op.apply(10, 0)
t0 = time.perf_counter(); r = op.apply(nt, 10); t1 = time.perf_counter()
print(f"plain     : device {r.device_seconds*1e3:8.2f} ms  wall {(t1-t0)*1e3:8.2f} ms")
op2 = P.Operator(prob)
op2.apply(10, 0)
t0 = time.perf_counter(); r2, snaps = op2.apply_snapshots(nt, every, 10, out=bufs); t1 = time.perf_counter()
gb = len(snaps) * n ** 3 * 4 / 1e9
print(f"snapshots : device {r2.device_seconds*1e3:8.2f} ms  wall {(t1-t0)*1e3:8.2f} ms  "
      f"({len(snaps)} x {n}^3 = {gb:.2f} GB drained, {gb/(t1-t0):.1f} GB/s of wall)")
