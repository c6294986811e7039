"""K3 vs K1 difference locator (development)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

so = int(sys.argv[1]) if len(sys.argv) > 1 else 12
shape = tuple(int(v) for v in sys.argv[2].split(',')) if len(sys.argv) > 2 else (46, 40, 75)
for nt in (2, 3, 4, 7):
    rng = np.random.default_rng(5)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    src = [shape[0] // 2 + 1, shape[1] // 2, shape[2] // 2 - 1]
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                                                   velocity_field=vel, damp_max=0.05, damp_width=4, source_point=src))
    rng = np.random.default_rng(so)
    init = [(rng.standard_normal(shape) * 1e-3).astype(np.float32) for _ in range(3)]
    outs = []
    for tb in (1, 2, 2):
        op = P.Operator(prob, time_block=tb)
        for l in range(3):
            op.set_level(l, init[l])
        op.apply(nt, 0)
        outs.append(op.levels())
        op.close()
    a, b, c = outs
    print(f"so={so} nt={nt} K3 deterministic={np.array_equal(b, c)} equal_K1={np.array_equal(a, b)}")
    for l in range(3):
        d = np.argwhere(a[l] != b[l])
        if len(d):
            xs = np.unique(d[:, 0])
            print(f"  level {l}: {len(d)} diffs, planes {xs.tolist()[:20]}, y {np.unique(d[:,1]).tolist()[:10]}.. z {np.unique(d[:,2]).tolist()[:10]}..")
