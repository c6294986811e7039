"""Stress of the fused in-kernel halo ordering at realistic sizes (development): P linked
z-slabs on disjoint SM partitions of one B200 (SWB_FUSED_SAME_DEVICE, SWB_MAX_CTAS = 148/P),
random initial levels, hundreds of steps; the final levels and per-step max must equal one
domain bit for bit.  Usage: python scripts/stress_fused.py [reps]"""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
from paper_1912_00695_b200 import dist as D

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rng = np.random.default_rng(2024)
bad = 0
for rep in range(reps):
    nslab = int(rng.integers(2, 5))
    so = int(rng.choice([4, 8, 12, 16]))
    n1, n2 = int(rng.integers(96, 200)), int(rng.integers(96, 200))
    n0 = nslab * int(rng.integers(40, 90))
    nt = int(rng.integers(100, 301))
    shape = (n0, n1, n2)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                   steps=nt, damp_max=0.02, damp_width=6))
    init = [(rng.standard_normal(shape) * 1e-3).astype(np.float32) for _ in range(3)]
    os.environ.pop("SWB_FUSED_SAME_DEVICE", None)
    os.environ.pop("SWB_MAX_CTAS", None)
    whole = P.Operator(prob)
    for l in range(3):
        whole.set_level(l, init[l])
    wr = whole.apply(nt, 0)
    ref = whole.levels().copy()
    whole.close()
    os.environ["SWB_FUSED_SAME_DEVICE"] = "1"
    os.environ["SWB_MAX_CTAS"] = str(148 // nslab)
    ops = [P.Operator(prob, slab=D.slab_bounds(n0, nslab, r)) for r in range(nslab)]
    for o in ops:
        for l in range(3):
            o.set_level(l, init[l])
    for lo, hi in zip(ops[:-1], ops[1:]):
        P.Operator.link_local(lo, hi)
    for o in ops:
        o.apply_async(nt, 0)
    smax = np.max([o.collect(nt) for o in ops], axis=0)
    fused = all(o.stats().kernel_launches == nt for o in ops)
    ok = np.array_equal(smax, wr.step_max_abs)
    for l in range(3):
        full = np.zeros(shape, np.float32)
        for o in ops:
            a, b = o.slab
            full[a:b] = o.get_level(l)[a:b]
        ok = ok and np.array_equal(full, ref[l])
    for o in ops:
        o.close()
    bad += not ok
    print(f"rep {rep}: {nslab} slabs, SO {so}, {shape}, {nt} steps, fused={fused}: {'OK' if ok else 'MISMATCH'}",
          flush=True)
print("STRESS_OK" if bad == 0 else f"STRESS_FAIL {bad}")
