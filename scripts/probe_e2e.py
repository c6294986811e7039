"""Breakdown of the end-to-end (public API, host buffers) time at 256^3 SO 8 (development)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

n, so, K = 256, 8, int(sys.argv[1]) if len(sys.argv) > 1 else 1000
shape = (n, n, n)
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=K + 8))
pin = lambda: torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()
m, damp = pin(), pin()
m[...] = prob.m_data(); damp[...] = prob.damp_data()
init = [pin() for _ in range(3)]
for a in init: a[...] = 0
out = [pin() for _ in range(3)]
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    op = P.Operator(prob, form="factorised", m=m, damp=damp); t.append(time.perf_counter())
    for l in range(3): op.set_level(l, init[l])
    t.append(time.perf_counter())
    r = op.apply(K, 0); t.append(time.perf_counter())
    for l in range(3): op.get_level(l, out[l])
    t.append(time.perf_counter())
    op.close(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: create {d[0]:.2f} ms, set_level x3 {d[1]:.2f}, apply {d[2]:.2f} (device {r.device_seconds*1e3:.2f}), "
          f"get_level x3 {d[3]:.2f}, close {d[4]:.2f}; e2e (create..get) {(t[4]-t[0])*1e3:.2f} ms")
