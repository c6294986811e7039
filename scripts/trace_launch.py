"""Per-CTA timeline of two back-to-back K1 launches (SWB_TRACE=1): python scripts/trace_launch.py SO n.

Stamps per CTA (globaltimer, ns): entry, after griddepcontrol.wait, warm-up done, consumers done,
exit.  Times are relative to the earliest entry of the first of the two launches, so the step
boundary shows as the gap between the last exit of step t and the waits of step t+1."""
import ctypes as C
import os
import sys

os.environ['SWB_TRACE'] = '1'
sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_1912_00695_b200 as P  # noqa: E402
from paper_1912_00695_b200 import _native as N  # noqa: E402

so = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=80))
op = P.Operator(prob)
op.apply(20, 0)
r = op.apply(40, 20)  # steps 20..59: the last two launches are steps 58 (even) and 59 (odd)
per_step = r.device_seconds / 40 * 1e6
buf = (C.c_uint64 * (2 * 8 * 1024))()
g = N.lib.swb_debug_trace(op._h, buf, 1024)
a = np.array(buf[:], dtype=np.float64).reshape(2, 1024, 8)[:, :g, :5]
t0 = a[0, :, 0].min()
a = (a - t0) / 1e3
print(f"SO {so} n {n}: {per_step:.1f} us/step over 40 back-to-back steps, CTAs {g}")
for s, name in ((0, "step t  "), (1, "step t+1")):
    e, w, wu, cd, ex = (a[s, :, i] for i in range(5))
    print(f"  {name}: entry {e.min():7.2f}..{e.max():7.2f}  wait done {w.min():7.2f}..{w.max():7.2f}  "
          f"warm-up done med {np.median(wu):7.2f}  compute done {cd.min():7.2f}/{np.median(cd):7.2f}/{cd.max():7.2f}  "
          f"exit {ex.min():7.2f}..{ex.max():7.2f}")
print(f"  boundary: last exit of t {a[0, :, 4].max():.2f} -> first wait done of t+1 {a[1, :, 1].min():.2f} "
      f"(gap {a[1, :, 1].min() - a[0, :, 4].max():.2f} us); step period {a[1, :, 1].min() - a[0, :, 1].min():.2f} us")
busy = (a[0, :, 3] - a[0, :, 1])
print(f"  stream time per CTA (wait done -> compute done) med {np.median(busy):.2f}, mean {busy.mean():.2f}, "
      f"max {busy.max():.2f}; SM-time busy fraction over the period "
      f"{busy.sum() / (148 * (a[1, :, 1].min() - a[0, :, 1].min())):.3f}")
op.close()
# per-CTA detail of step t: stream time against the SM id and the item (column, chunk)
raw = np.array(buf[:], dtype=np.float64).reshape(2, 1024, 8)[0, :g]
sm = raw[:, 5].astype(int)
st = (raw[:, 3] - raw[:, 1]) / 1e3
NCOL, NZT = int(os.environ.get("TRACE_NCOL", "36")), int(os.environ.get("TRACE_NZT", "4"))
if os.environ.get("TRACE_DETAIL"):
    order = np.argsort(st)
    print("  fastest 6 (cta, sm, us):", [(int(b), int(sm[b]), round(float(st[b]), 2)) for b in order[:6]])
    print("  slowest 6 (cta, sm, us):", [(int(b), int(sm[b]), round(float(st[b]), 2)) for b in order[-6:]])
    for name, key in (("sm // 2 (TPC) parity", lambda b: (sm[b] // 2) % 2), ("sm < 74", lambda b: int(sm[b] < 74)),
                      ("sm % 4", lambda b: sm[b] % 4),
                      # items = CTAs here (one item each): item = chunk * ncol + col, col = ytile * nzt + ztile
                      ("chunk", lambda b: b // NCOL), ("z tile", lambda b: (b % NCOL) % NZT),
                      ("y tile", lambda b: (b % NCOL) // NZT)):
        grp = {}
        for b in range(g):
            grp.setdefault(key(b), []).append(st[b])
        print(f"  by {name}: " + "  ".join(f"{k}:{np.mean(v):.2f}" for k, v in sorted(grp.items())))
    np.save("gpurun_out/trace_detail_%d_%d.npy" % (so, n), raw)
