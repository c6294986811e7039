"""Per-CTA timeline of one stencil launch (SWB_TRACE=1)."""
import ctypes as C, os, sys
os.environ['SWB_TRACE'] = '1'
sys.path.insert(0, '.')
import numpy as np
import paper_1912_00695_b200 as P
from paper_1912_00695_b200 import _native as N
so = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=40))
op = P.Operator(prob)
op.apply(20, 0)
r = op.apply(1, 20)
buf = (C.c_uint64 * (4 * 1024))()
g = N.lib.swb_debug_trace(op._h, buf, 1024)
t = np.array(buf[:4 * g], dtype=np.float64).reshape(g, 4)
t0 = t[:, 0].min()
t = (t - t0) / 1e3
print(f"SO {so} n {n}: launch {r.device_seconds*1e6:.1f} us (event), CTAs {g}")
print(f"  start   : min {t[:,0].min():7.2f} max {t[:,0].max():7.2f} us")
print(f"  warm-up : min {t[:,1].min():7.2f} med {np.median(t[:,1]):7.2f} max {t[:,1].max():7.2f} us")
print(f"  compute : min {t[:,2].min():7.2f} med {np.median(t[:,2]):7.2f} max {t[:,2].max():7.2f} us")
print(f"  exit    : min {t[:,3].min():7.2f} med {np.median(t[:,3]):7.2f} max {t[:,3].max():7.2f} us")
# correlate with the item geometry (one item per CTA when grid == items)
ny = n - so; nzt = -(-(n - so // 2 - (so // 2 & ~3)) // 64)
import math
T1 = int(os.environ.get("T1", "30" if so <= 12 else "22"))
nyt = -(-ny // T1); ncol = nyt * nzt
nch = g // ncol if g % ncol == 0 else None
print(f"  ncol={ncol} (nyt={nyt}, nzt={nzt}) nchunk={nch}")
if nch:
    dur = t[:, 2] - t[:, 1]
    for name, key in (("z-tile", lambda b: (b % ncol) % nzt), ("y-tile", lambda b: (b % ncol) // nzt),
                      ("chunk", lambda b: b // ncol)):
        groups = {}
        for b in range(g):
            groups.setdefault(key(b), []).append(dur[b])
        print(f"  by {name}: " + "  ".join(f"{k}:{np.mean(v):.1f}" for k, v in sorted(groups.items())))
    print("  slowest 8 CTAs (b, col, chunk, us):", [(int(b), int(b % ncol), int(b // ncol), round(float(dur[b]), 1)) for b in np.argsort(-dur)[:8]])
