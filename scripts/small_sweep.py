"""Small grids: K1 step cost with the plan's dim-0 chunk count against forced counts (SWB_NCHUNK),
and the one-thread-per-point factorised kernel.  python scripts/small_sweep.py [n:so ...]"""
import os
import sys
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]] or [(64, 2)]
for n, so in cases:
    nt = 200
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n,) * 3, spacing=(10., 10., 10.), space_order=so,
                                                   steps=nt + 20))
    for nc in ["", "16", "24", "32", "40", "49", "56", "64"]:
        if nc:
            os.environ["SWB_NCHUNK"] = nc
        else:
            os.environ.pop("SWB_NCHUNK", None)
        op = P.Operator(prob)
        op.apply(10, 0)
        t = op.apply(nt, 10).device_seconds / nt * 1e6
        print(f"n {n} SO {so:2d} K1 nchunk {nc or 'plan'}: {t:.2f} us/step", flush=True)
        op.close()
    os.environ.pop("SWB_NCHUNK", None)
    op = P.Operator(prob, form="factorised_simple")
    op.apply(10, 0)
    print(f"n {n} SO {so:2d} factorised_simple: {op.apply(nt, 10).device_seconds / nt * 1e6:.2f} us/step")
    op.close()
