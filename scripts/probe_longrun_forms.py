"""Long-run FP32 error of the factorised kernels against the bit-exact FP64 kernel (development).
Which part drifts: K1 (FP32 combine with the B = 1/(m+g), A coefficient fields), the
one-thread-per-point factorised form with an FP64 combine (factorised_simple), and with K1's
FP32 combine (factorised_simple_f32c).  Two media: constant velocity undamped (the bench
workload's medium) and a random heterogeneous damped one.
  python scripts/probe_longrun_forms.py [n] [so ...]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sos = [int(x) for x in sys.argv[2:]] or [4, 8, 16]
marks = [1000, 3000, 10000]
forms = ("factorised", "factorised_simple", "factorised_simple_f32c")
for so in sos:
    for medium in ("constant", "hetero-damped"):
        rng = np.random.default_rng(so)
        shape = (n, n, n)
        if medium == "constant":
            cfg = P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=marks[-1])
        else:
            vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
            cfg = P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=marks[-1],
                                      velocity_field=vel, damp_max=0.05, damp_width=10)
        prob = P.make_wave_problem(cfg)
        ex = P.Operator(prob, form="plain_f64")
        ops = {f: P.Operator(prob, form=f) for f in forms}
        done = 0
        for m in marks:
            ex.apply(m - done, done)
            for o in ops.values():
                o.apply(m - done, done)
            done = m
            y = ex.get_level(m % 3).astype(np.float64)
            errs = {f: f"{np.linalg.norm(o.get_level(m % 3) - y) / np.linalg.norm(y):.2e}" for f, o in ops.items()}
            print(f"SO {so:2d} {medium:14s} step {m:6d}", errs, flush=True)
        for o in list(ops.values()) + [ex]:
            o.close()
