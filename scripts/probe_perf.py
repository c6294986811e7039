"""Quick device-time probe of each stencil form at 256^3 (not the bench; for development)."""
import os, sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

forms = sys.argv[1].split(',') if len(sys.argv) > 1 else ['factorised_simple', 'plain_f64', 'plain_f32']
sos = [int(s) for s in sys.argv[2].split(',')] if len(sys.argv) > 2 else [4, 8, 12, 16]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 256
nt = int(sys.argv[4]) if len(sys.argv) > 4 else 50
for so in sos:
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so, steps=nt + 10))
    pts = (n - so) ** 3
    for f in forms:
        op = P.Operator(prob, form=f, time_block=int(os.environ.get("TB", "1")))
        op.apply(5, 0)
        r = op.apply(nt, 5)
        st = op.stats()
        gpts = pts * nt / r.device_seconds / 1e9
        print(f"so={so:2d} form={f:18s} variant={st.kernel_variant} {r.device_seconds / nt * 1e6:9.1f} us/step  {gpts:7.1f} GPts/s  {20 * gpts / 6534.1 * 100:5.1f}% HBM-roofline(20B/pt)", flush=True)
        op.close()
