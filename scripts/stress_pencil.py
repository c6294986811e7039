"""Stress: many seeded random SO 16 problems on the y-pencil K1 variant (forced with SWB_YW=1,
SWB_T1=20) against the C restatement (<= 1e-5), plus fused z-slab decompositions bitwise equal to
one domain.  python scripts/stress_pencil.py [n_cases]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SWB_YW"], os.environ["SWB_T1"] = "1", "20"
import paper_1912_00695_b200 as P  # noqa: E402
from oracle import bindings as O  # noqa: E402

ncase = int(sys.argv[1]) if len(sys.argv) > 1 else 100
worst, fails = 0.0, 0
for seed in range(ncase):
    rng = np.random.default_rng(90000 + seed)
    so, h = 16, 8
    shape = tuple(int(rng.integers(2 * h + 3, 2 * h + 70)) for _ in range(3))
    nt = int(rng.integers(2, 30))
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    damp, width = float(rng.choice([0.0, 0.03, 0.1])), int(rng.integers(1, 8))
    src = [int(rng.integers(h, s - h)) for s in shape]
    init = [(rng.standard_normal(shape) * 1e-2).astype(np.float32) for _ in range(3)]
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                                                   velocity_field=vel, damp_max=damp, damp_width=width, source_point=src))
    ref = O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=nt, velocity_field=vel, damp_max=damp,
                                    damp_width=width, source_point=src), initial_u=init)
    op = P.Operator(prob)
    assert op.stats().kernel_variant // 10000000 == 1
    for l in range(3):
        op.set_level(l, init[l])
    op.apply(nt, 0)
    fl = nt % 3
    a, b = op.get_level(fl).astype(np.float64), ref["levels"][fl].astype(np.float64)
    err = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
    worst = max(worst, err)
    ok = err <= 1e-5
    if shape[0] >= 4 * h and seed % 3 == 0:  # fused slabs, bitwise against the single domain
        whole = op.get_level(fl)
        os.environ["SWB_FUSED_SAME_DEVICE"], os.environ["SWB_MAX_CTAS"] = "1", "74"
        cut = int(rng.integers(h, shape[0] - h))
        ops = [P.Operator(prob, slab=s) for s in ((0, cut), (cut, shape[0]))]
        P.Operator.link_local(ops[0], ops[1])
        for o in ops:
            for l in range(3):
                o.set_level(l, init[l])
        for o in ops:
            o.apply_async(nt, 0)
        for o in ops:
            o.collect(nt)
        full = np.concatenate([ops[0].get_level(fl)[:cut], ops[1].get_level(fl)[cut:]])
        ok &= bool(np.array_equal(full, whole))
        for o in ops:
            o.close()
        del os.environ["SWB_FUSED_SAME_DEVICE"], os.environ["SWB_MAX_CTAS"]
    op.close()
    fails += 0 if ok else 1
    if not ok:
        print("FAIL", seed, shape, nt, err, flush=True)
print(f"pencil stress: {ncase} cases, {fails} failures, worst rel L2 {worst:.2e}", flush=True)
