"""Hash of K1 results over a set of problems (development: bitwise A/B of two builds via SWB_LIB)."""
import hashlib, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
h = hashlib.sha256()
for so in (2, 4, 6, 8, 10, 12, 16):
    for shape, damp in (((40, 44, 70), 0.0), ((37, 29, 53), 0.05), ((96, 96, 96), 0.02)):
        rng = np.random.default_rng(so)
        vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
        prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                       steps=23, velocity_field=vel, damp_max=damp,
                                                       damp_width=5))
        op = P.Operator(prob)
        init = [(rng.standard_normal(shape) * 1e-3).astype(np.float32) for _ in range(3)]
        for l in range(3):
            op.set_level(l, init[l])
        r = op.apply(23, 0)
        h.update(op.levels().tobytes())
        h.update(np.asarray(r.step_max_abs).tobytes())
        op.close()
print(h.hexdigest())
