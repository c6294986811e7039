"""Compare the factorised kernel variants against the bit-exact plain-FP64 kernel on small
shapes (development check)."""
import os, sys
import numpy as np
sys.path.insert(0, '.')
import paper_1912_00695_b200 as P
cases = [((16, 17, 18), 2, 11, 0.0), ((24, 26, 28), 8, 20, 0.05), ((30, 31, 32), 16, 11, 0.0),
         ((40, 50, 70), 4, 9, 0.0), ((64, 64, 64), 2, 30, 0.0), ((20, 21, 22), 12, 6, 0.02)]
for shape, so, nt, damp in cases:
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=so, steps=nt,
                                                   damp_max=damp, damp_width=4))
    ref = P.Operator(prob, form='plain_f64'); ref.apply(nt, 0); R = ref.levels()
    line = []
    for kern in ('sq', 'rq'):
        os.environ['SWB_KERNEL'] = kern
        op = P.Operator(prob, form='factorised'); op.apply(nt, 0); L = op.levels()
        fl = nt % 3
        e = np.linalg.norm(L[fl] - R[fl]) / np.linalg.norm(R[fl])
        bad = np.argwhere(np.abs(L[fl] - R[fl]) > 1e-3 * np.abs(R[fl]).max())
        line.append(f"{kern}: var={op.stats().kernel_variant} err={e:.2e} nbad={len(bad)} first={bad[:3].tolist()}")
    print(shape, so, nt, damp, ' | '.join(line), flush=True)
