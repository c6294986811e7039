"""Relative L2 of each FP32 form vs the bit-exact plain-FP64 kernel (== reference
interpreter) after nt steps.  Development probe."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
damp = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
sos = [int(s) for s in sys.argv[4].split(',')] if len(sys.argv) > 4 else [4, 8, 12, 16]
forms = sys.argv[5].split(',') if len(sys.argv) > 5 else ['factorised', 'factorised_simple', 'factorised_simple_f32c', 'plain_f32']
for so in sos:
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n, n, n), spacing=(10., 10., 10.), space_order=so,
                                                   steps=nt, damp_max=damp, damp_width=10))
    ref = P.Operator(prob, form='plain_f64')
    rr = ref.apply(nt, 0)
    R = ref.levels()
    fl = nt % 3
    line = []
    for f in forms:
        op = P.Operator(prob, form=f)
        r = op.apply(nt, 0)
        L = op.levels()
        e = np.linalg.norm((L[fl] - R[fl]).astype(np.float64)) / np.linalg.norm(R[fl].astype(np.float64))
        em = np.max(np.abs(r.step_max_abs - rr.step_max_abs) / np.maximum(rr.step_max_abs, 1e-30))
        line.append(f"{f}={e:.2e}(smax {em:.1e})")
        op.close()
    print(f"n={n} nt={nt} damp={damp} so={so}: " + "  ".join(line), flush=True)
