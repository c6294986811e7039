"""SO 4 long-run error: which part of the FP32 combine drifts (development)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
n, so = 96, 4
marks = [1000, 3000, 10000]
rng = np.random.default_rng(so)
shape = (n, n, n)
vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=marks[-1],
                                               velocity_field=vel, damp_max=0.05, damp_width=10))
ex = P.Operator(prob, form="plain_f64")
ops = {f: P.Operator(prob, form=f) for f in ("factorised", "factorised_simple", "factorised_simple_f32c")}
done = 0
for m in marks:
    ex.apply(m - done, done)
    for o in ops.values():
        o.apply(m - done, done)
    done = m
    y = ex.get_level(m % 3).astype(np.float64)
    print(m, {f: f"{np.linalg.norm(o.get_level(m % 3) - y) / np.linalg.norm(y):.2e}" for f, o in ops.items()}, flush=True)
