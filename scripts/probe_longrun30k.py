"""K1 (factorised FP32) against the bit-exact FP64 kernel out to the paper's 30,000-step timing
protocol: relative L2 of the newest level at 1k/10k/20k/30k steps, 128^3,
constant undamped and heterogeneous damped media.  python scripts/probe_longrun30k.py [so ...]"""
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_1912_00695_b200 as P  # noqa: E402

n = 128
sos = [int(x) for x in sys.argv[1:]] or [4, 8, 12, 16]
marks = [1000, 10000, 20000, 30000]
for so in sos:
    for medium in ("constant", "hetero-damped"):
        shape = (n, n, n)
        kw = {}
        if medium != "constant":
            rng = np.random.default_rng(so)
            kw = dict(velocity_field=(1500 + 1500 * rng.random(shape)).astype(np.float32), damp_max=0.05,
                      damp_width=10)
        prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                       steps=marks[-1], **kw))
        ex, k1 = P.Operator(prob, form="plain_f64"), P.Operator(prob)
        done, out = 0, []
        for m in marks:
            ex.apply(m - done, done)
            k1.apply(m - done, done)
            done = m
            y = ex.get_level(m % 3).astype(np.float64)
            out.append(f"{m}: {np.linalg.norm(k1.get_level(m % 3) - y) / np.linalg.norm(y):.2e}")
        print(f"SO {so:2d} {medium:14s} variant {k1.stats().kernel_variant}  " + "  ".join(out), flush=True)
        ex.close()
        k1.close()
