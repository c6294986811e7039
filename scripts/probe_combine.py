"""K1 combine variants (development; SWB_LIB selects the build): long-run error of K1 against the
bit-exact FP64 kernel, and K1 throughput at 256^3.
  SWB_LIB=paper_1912_00695_b200/_lib/variants/libswb_combine2.so python scripts/probe_combine.py"""
import os
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

lib = os.path.basename(os.environ.get("SWB_LIB", "libswb.so"))
n = 128
marks = [1000, 3000, 10000]
for so in (4, 8, 16):
    for medium in ("constant", "hetero-damped"):
        rng = np.random.default_rng(so)
        shape = (n, n, n)
        kw = {}
        if medium != "constant":
            kw = dict(velocity_field=(1500 + 1500 * rng.random(shape)).astype(np.float32), damp_max=0.05,
                      damp_width=10)
        prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                       steps=marks[-1], **kw))
        ex, k1 = P.Operator(prob, form="plain_f64"), P.Operator(prob)
        done, errs = 0, []
        for m in marks:
            ex.apply(m - done, done)
            k1.apply(m - done, done)
            done = m
            y = ex.get_level(m % 3).astype(np.float64)
            errs.append(f"{np.linalg.norm(k1.get_level(m % 3) - y) / np.linalg.norm(y):.2e}")
        print(f"{lib} SO {so:2d} {medium:14s} err@1k/3k/10k {' '.join(errs)}", flush=True)
        ex.close()
        k1.close()
for so in (4, 8, 12, 16):
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(256,) * 3, spacing=(10., 10., 10.), space_order=so,
                                                   steps=420))
    op = P.Operator(prob)
    op.apply(10, 0)
    best = 0
    for rep in range(3):
        r = op.apply(100, 10 + 100 * rep)
        best = max(best, (256 - so) ** 3 * 100 / r.device_seconds / 1e9)
    print(f"{lib} SO {so:2d} 256^3 K1 {best:.1f} GPts/s", flush=True)
    op.close()
