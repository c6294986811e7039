"""Small-grid (config 1: 64^3 SO 2, 100 steps) per-step cost, with and without the receiver line."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
shape, so, nt = (64, 64, 64), 2, 100
prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt + 10))
rec = np.array([[32, 40, z] for z in range(1, 63)], np.int32)
for tag, kw in (("no receivers", {}), ("receiver line", {"receivers": rec})):
    for form in ("factorised", "plain_f64"):
        op = P.Operator(prob, form=form, **kw)
        op.apply(10, 0)
        r = op.apply(nt, 10)
        print(f"{tag:14s} {form:11s}: {r.device_seconds / nt * 1e6:6.2f} us/step  {62**3 * nt / r.device_seconds / 1e9:6.2f} GPts/s  launches {op.stats().kernel_launches}")
# kernel choice at small grids: the one-thread-per-point factorised kernel vs K1
for form in ("factorised_simple",):
    op = P.Operator(prob, form=form)
    op.apply(10, 0)
    r = op.apply(nt, 10)
    print(f"no receivers   {form:11s}: {r.device_seconds / nt * 1e6:6.2f} us/step  {62**3 * nt / r.device_seconds / 1e9:6.2f} GPts/s")
