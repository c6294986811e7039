"""Cost of the fused z-slab halo exchange, measured on ONE B200: the grid split into P
linked slabs that run concurrently on P disjoint SM partitions (SWB_MAX_CTAS = 148/P,
in-kernel neighbour waits + peer stores, SWB_FUSED_SAME_DEVICE), against one domain
on all 148 SMs.  Same device memory, so this isolates the synchronisation/ordering cost of the
exchange (not NVLink bandwidth).  Development/report script."""
import os, sys, time
import numpy as np
sys.path.insert(0, '.')
P_SLABS = int(sys.argv[1]) if len(sys.argv) > 1 else 2
so = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256
nt = int(sys.argv[4]) if len(sys.argv) > 4 else 200
os.environ["SWB_FUSED_SAME_DEVICE"] = "1"
import paper_1912_00695_b200 as P
from paper_1912_00695_b200 import dist as D

shape = (n * P_SLABS, n, n)
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt + 20))
pts = (shape[0] - so) * (n - so) ** 2
os.environ["SWB_MAX_CTAS"] = str(148 // P_SLABS)
ops = [P.Operator(prob, slab=D.slab_bounds(shape[0], P_SLABS, r)) for r in range(P_SLABS)]
for lo, hi in zip(ops[:-1], ops[1:]):
    P.Operator.link_local(lo, hi)
for o in ops:
    o.apply_async(5, 0)
for o in ops:
    o.collect(5)
t0 = time.perf_counter()
for o in ops:
    o.apply_async(nt, 5)
for o in ops:
    o.collect(nt)
wall = time.perf_counter() - t0
dev = max(o.stats().device_ms for o in ops) * 1e-3
print(f"{P_SLABS} linked slabs x {148 // P_SLABS} SMs: {pts * nt / dev / 1e9:7.1f} GPts/s (device max), {pts * nt / wall / 1e9:7.1f} (wall)")
for o in ops:
    o.close()
# the same partitioning without any exchange: P independent n^3 domains, concurrently, each
# capped at 148/P CTAs (isolates the cost of splitting the SMs from the cost of the exchange)
sub = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=nt + 20))
ind = [P.Operator(sub) for _ in range(P_SLABS)]
for o in ind:
    o.apply_async(5, 0)
for o in ind:
    o.collect(5)
for o in ind:
    o.apply_async(nt, 5)
for o in ind:
    o.collect(nt)
dev2 = max(o.stats().device_ms for o in ind) * 1e-3
pts2 = P_SLABS * (n - so) ** 3
print(f"{P_SLABS} independent {n}^3 x {148 // P_SLABS} SMs: {pts2 * nt / dev2 / 1e9:7.1f} GPts/s (no exchange)")
for o in ind:
    o.close()
os.environ.pop("SWB_MAX_CTAS")
# reference: the same global grid as one domain on all SMs, and as P independent slab-sized
# domains each on its SM share
one = P.Operator(prob)
one.apply(5, 0)
r = one.apply(nt, 5)
print(f"1 domain x 148 SMs   : {pts * nt / r.device_seconds / 1e9:7.1f} GPts/s")
one.close()
