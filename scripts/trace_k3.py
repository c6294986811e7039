"""Per-CTA timeline of one K3 (time_block=2) launch (SWB_TRACE=1): stage-1 vs stage-2 CTAs."""
import ctypes as C, os, sys
os.environ['SWB_TRACE'] = '1'
sys.path.insert(0, '.')
import numpy as np
import paper_1912_00695_b200 as P
from paper_1912_00695_b200 import _native as N
so = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=40))
op = P.Operator(prob, time_block=2)
op.apply(20, 0)
r = op.apply(2, 20)
buf = (C.c_uint64 * (4 * 1024))()
g = N.lib.swb_debug_trace(op._h, buf, 1024)
t = np.array(buf[:4 * g], dtype=np.float64).reshape(g, 4)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
print(f"K3 SO {so} n {n}: launch {r.device_seconds*1e6:.1f} us (event), CTAs {g}")
half = g // 2
for name, sl in (("stage1", slice(0, half)), ("stage2", slice(half, g))):
    u = t[sl]
    print(f" {name}: start {u[:,0].min():6.1f}-{u[:,0].max():6.1f}  warm-up med {np.median(u[:,1]):6.1f} max {u[:,1].max():6.1f}"
          f"  compute med {np.median(u[:,2]):6.1f} max {u[:,2].max():6.1f}  exit max {u[:,3].max():6.1f} us")
