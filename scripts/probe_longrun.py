"""Error growth of the FP32 factorised kernel (K1) against the bit-exact plain FP64 kernel (which
equals the reference interpreter) over long runs (development/report script)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
marks = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1000", "2000", "5000", "10000"])]
for so in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4", "8", "16"])]:
    rng = np.random.default_rng(so)
    shape = (n, n, n)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so,
                                                   steps=marks[-1], velocity_field=vel, damp_max=0.05,
                                                   damp_width=10))
    a = P.Operator(prob)                    # factorised, FP32 (K1)
    b = P.Operator(prob, form="plain_f64")  # bit-exact with the reference interpreter
    done, out = 0, []
    for m in marks:
        a.apply(m - done, done)
        b.apply(m - done, done)
        done = m
        l = m % 3
        x, y = a.get_level(l).astype(np.float64), b.get_level(l).astype(np.float64)
        out.append(f"{m}: {np.linalg.norm(x - y) / np.linalg.norm(y):.2e}")
    print(f"{n}^3 SO {so:2d} damped heterogeneous, rel L2 K1 vs exact after " + ", ".join(out), flush=True)
