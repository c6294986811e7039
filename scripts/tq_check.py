"""TMEM-queue K1 variants (SWB_UNR=0) against the register-queue K1: bitwise equality and speed."""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, '.')
code = r'''
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
so, n, nt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(so)
shape = (n, n + 2, n + 6)
vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt,
                                               velocity_field=vel, damp_max=0.05, damp_width=5))
op = P.Operator(prob)
r = op.apply(nt, 0)
np.save(sys.argv[4], op.levels())
print(op.stats().kernel_variant, r.step_max_abs[-1])
'''
for so, t1 in ((16, "30"), (16, "22"), (12, "30")):
    outs = []
    for unr in ("", "0"):
        env = dict(os.environ)
        if unr:
            env["SWB_UNR"] = unr
            env["SWB_T1"] = t1
        f = f"/tmp/tq_{so}_{unr or 'k1'}.npy"
        pr = subprocess.run([sys.executable, "-c", code, str(so), "70", "20", f], env=env, capture_output=True, text=True)
        print(so, t1, unr or "k1", pr.stdout.strip(), pr.stderr.strip()[-300:])
        outs.append(np.load(f) if os.path.exists(f) else None)
    if outs[0] is not None and outs[1] is not None:
        print(f"  SO {so} T1 {t1}: TMEM queue == register queue bitwise: {np.array_equal(outs[0], outs[1])}")
