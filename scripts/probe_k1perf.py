"""K1 device throughput at 256^3 (SO 4/8/12/16) and 512^3 SO 8 (development A/B: run under
different SWB_LIB builds / SWB_* switches).  Best of 3 x 100 steps after warm-up."""
import os
import sys
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

tag = os.environ.get("TAG", os.path.basename(os.environ.get("SWB_LIB", "libswb.so")))
cases = [(256, s) for s in (4, 8, 12, 16)] + [(512, 8)]
if len(sys.argv) > 1:
    cases = [tuple(int(v) for v in a.split(":")) for a in sys.argv[1:]]
for n, so in cases:
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n,) * 3, spacing=(10., 10., 10.), space_order=so,
                                                   steps=420))
    op = P.Operator(prob)
    op.apply(10, 0)
    best = 0
    for rep in range(3):
        r = op.apply(100, 10 + 100 * rep)
        best = max(best, (n - so) ** 3 * 100 / r.device_seconds / 1e9)
    print(f"{tag} n {n} SO {so:2d} K1 {best:.1f} GPts/s", flush=True)
    op.close()
