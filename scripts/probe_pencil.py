"""A/B of the K1 y-pencil variants (SWB_YW / SWB_T1 / SWB_UNR switches, read per handle):
accuracy against the bit-exact basic kernel on a damped heterogeneous 96^3 problem, and
device throughput (best of 3 x 100 steps) at the sizes given as n:so[:T1:YW[:UNR]]."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
import paper_1912_00695_b200 as P  # noqa: E402


def setenv(t1, yw, unr):
    for k, v in (("SWB_T1", t1), ("SWB_YW", yw), ("SWB_UNR", unr)):
        if v:
            os.environ[k] = str(v)
        else:
            os.environ.pop(k, None)


def accuracy(so, t1, yw, unr, n=96, nt=60):
    shape = (n, n + 4, n + 8)
    rng = np.random.default_rng(3)
    vel = (1500.0 + 1500.0 * rng.random(shape)).astype(np.float32)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt,
                                                   velocity_field=vel, damp_max=0.05, damp_width=6))
    setenv(0, 0, 0)
    exact = P.run(prob, dse=P.DseLevel.basic)
    setenv(t1, yw, unr)
    fast = P.run(prob, dse=P.DseLevel.aggressive)
    fl = fast.final_level
    a, b = fast.u.data[fl].astype(np.float64), exact.u.data[fl].astype(np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b)), fast


def speed(n, so, t1, yw, unr):
    setenv(t1, yw, unr)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n,) * 3, spacing=(10., 10., 10.), space_order=so,
                                                   steps=420))
    op = P.Operator(prob)
    op.apply(10, 0)
    best = 0
    for rep in range(3):
        r = op.apply(100, 10 + 100 * rep)
        best = max(best, (n - so) ** 3 * 100 / r.device_seconds / 1e9)
    var = op.stats().kernel_variant if hasattr(op, "stats") else -1
    op.close()
    return best, var


for arg in sys.argv[1:]:
    f = [int(v) for v in arg.split(":")] + [0, 0, 0]
    n, so, t1, yw, unr = f[:5]
    err, _ = accuracy(so, t1, yw, unr)
    gp, var = speed(n, so, t1, yw, unr)
    print(f"n {n} SO {so:2d} T1 {t1} YW {yw} UNR {unr}: rel L2 {err:.2e}  {gp:.1f} GPts/s  variant {var}",
          flush=True)
