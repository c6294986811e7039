"""m and damp computed on the device (swb_problem.velocity / damp_max / damp_width with NULL m,
damp) are bit-identical to WaveProblem::m_data / damp_data computed on the host
(src/wave_model.cpp:16-45): the runs through both routes agree bit for bit, single domain and
z-slabs (the taper uses global plane coordinates)."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P

pytestmark = pytest.mark.gpu


def problem(shape, so, nt, damp_max, width):
    rng = np.random.default_rng(3)
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    return P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp_max,
                                                   damp_width=width))


@pytest.mark.parametrize("form", ["plain_f64", "factorised"])
@pytest.mark.parametrize("damp_max,width", [(0.05, 4), (0.0, 10), (0.05, 0), (2e-5, 10)])
def test_device_fields_equal_host_fields(form, damp_max, width):
    shape, so, nt = (30, 33, 36), 8, 14
    prob = problem(shape, so, nt, damp_max, width)
    rec = np.array([[15, y, 17] for y in range(shape[1])], np.int32)
    dev = P.Operator(prob, form=form, receivers=rec)  # velocity + taper parameters
    host = P.Operator(prob, form=form, receivers=rec, m=prob.m_data(), damp=prob.damp_data())
    a, b = dev.apply(nt, 0), host.apply(nt, 0)
    assert np.array_equal(dev.levels(), host.levels())
    assert np.array_equal(a.step_max_abs, b.step_max_abs) and np.array_equal(a.rec_traces, b.rec_traces)


def test_device_taper_on_slabs():
    shape, so, nt = (40, 26, 28), 4, 12
    prob = problem(shape, so, nt, 0.05, 5)
    one = P.Operator(prob, form="plain_f64", m=prob.m_data(), damp=prob.damp_data())
    one.apply(nt, 0)
    ref = one.levels()
    ops = [P.Operator(prob, form="plain_f64", slab=s) for s in ((0, 13), (13, 27), (27, 40))]
    P.Operator.link_local(ops[0], ops[1])
    P.Operator.link_local(ops[1], ops[2])
    for o in ops:
        o.apply_async(nt, 0)
    for o in ops:
        o.collect(nt)
    got = np.zeros_like(ref)
    for o in ops:
        lo, hi = o.slab
        got[:, lo:hi] = o.levels()[:, lo:hi]
    assert np.array_equal(got, ref)
