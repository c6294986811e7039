"""Coverage of the configuration space beyond the golden cases: every even space order the
C-ABI accepts (2..24; K1 variants exist up to SO 16, larger orders run the one-thread-per-point
kernels), anisotropic spacing (the factorised path without the isotropic TMA kernel), and odd,
non-cubic shapes down to the smallest grid each order allows.  Oracle: the C restatement."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P
from oracle import bindings as O

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _pair(shape, so, nt, spacing=(10.0, 10.0, 10.0), seed=1, damp=0.05):
    rng = np.random.default_rng(seed)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    cfg = P.WaveProblemConfig(shape=shape, spacing=spacing, space_order=so, steps=nt, velocity_field=vel,
                              damp_max=damp, damp_width=3)
    ocfg = O.OracleConfig(shape=shape, spacing=spacing, space_order=so, steps=nt, velocity_field=vel,
                          damp_max=damp, damp_width=3)
    return P.make_wave_problem(cfg), ocfg


@pytest.mark.parametrize("so", list(range(2, 26, 2)))
def test_every_space_order(so):
    shape, nt = (33, 30, 37), 25
    prob, ocfg = _pair(shape, so, nt)
    ref = O.port_run(ocfg)
    exact = P.run(prob, dse=P.DseLevel.basic)
    assert np.array_equal(exact.u.data, ref["levels"])
    assert np.array_equal(exact.step_max_abs, ref["step_max_abs"])
    fast = P.run(prob, dse=P.DseLevel.aggressive)
    fl = fast.final_level
    assert rel_l2(fast.u.data[fl], ref["levels"][fl]) <= 1e-5


@pytest.mark.parametrize("so", [4, 8, 16])
def test_anisotropic_spacing(so):
    shape, nt = (36, 34, 40), 30
    prob, ocfg = _pair(shape, so, nt, spacing=(10.0, 12.5, 15.0), seed=so)
    ref = O.port_run(ocfg)
    exact = P.run(prob, dse=P.DseLevel.basic)
    assert np.array_equal(exact.u.data, ref["levels"])
    fast = P.run(prob, dse=P.DseLevel.aggressive)
    fl = fast.final_level
    assert rel_l2(fast.u.data[fl], ref["levels"][fl]) <= 1e-5


@pytest.mark.parametrize("so", [2, 8, 16])
def test_smallest_grids(so):
    h = so // 2
    shape, nt = (2 * h + 1 + 2, 2 * h + 1 + 1, 2 * h + 1 + 3), 12  # a few updated points per axis
    prob, ocfg = _pair(shape, so, nt, damp=0.0)
    ref = O.port_run(ocfg)
    exact = P.run(prob, dse=P.DseLevel.basic)
    assert np.array_equal(exact.u.data, ref["levels"])
    fast = P.run(prob, dse=P.DseLevel.aggressive)
    fl = fast.final_level
    assert rel_l2(fast.u.data[fl], ref["levels"][fl]) <= 1e-5


def test_handles_recycled_through_the_buffer_pool():
    """Every device buffer of a handle (fields, counters, flags, traces) is recycled through the
    process-wide pool on destroy.  Interleaved handles of two problems and two forms, with
    receivers and damping, must reproduce their first results bit for bit on every reuse."""
    def make(shape, so, seed):
        rng = np.random.default_rng(seed)
        vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
        return P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                       steps=9, velocity_field=vel, damp_max=0.05,
                                                       damp_width=4))
    cases = [(make((36, 40, 70), 8, 1), "factorised"), (make((30, 34, 44), 4, 2), "factorised"),
             (make((36, 40, 70), 8, 1), "plain_f64")]
    first = {}
    for rnd in range(4):
        for ci, (prob, form) in enumerate(cases):
            rec = np.array([[x, 12, 20] for x in range(4, prob.shape[0] - 4, 5)], np.int32)
            op = P.Operator(prob, form=form, receivers=rec)
            r = op.apply(9, 0)
            got = (op.levels().copy(), np.asarray(r.step_max_abs).copy(), np.asarray(r.rec_traces).copy())
            op.close()
            if rnd == 0:
                first[ci] = got
            else:
                for a, b in zip(first[ci], got):
                    assert np.array_equal(a, b), (rnd, ci)
    # the two forms on the same problem agree to the north-star tolerance
    fl = 9 % 3
    assert rel_l2(first[0][0][fl], first[2][0][fl]) <= 1e-5
