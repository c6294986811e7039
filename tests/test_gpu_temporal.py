"""Temporal blocking (K3, time_block=2): two time steps per launch, stage-1 CTAs computing
u[t+1] (plus H dim-0 overlap planes per chunk side) and stage-2 CTAs computing u[t+2] from
it behind per-plane progress counters.  The per-point arithmetic is K1's, so the gate is
SURVEY §7 step 7: K3 final levels == K1 final levels bit for bit (and the per-step max|u|,
receiver traces and the instability step with them), for every space order, odd and even
step counts, several chunks and several items per CTA (grid capped with SWB_MAX_CTAS)."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P

pytestmark = pytest.mark.gpu


def _problem(shape, so, nt, seed=5, damp=0.05):
    rng = np.random.default_rng(seed)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    src = [shape[0] // 2 + 1, shape[1] // 2, shape[2] // 2 - 1]
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                              velocity_field=vel, damp_max=damp, damp_width=4, source_point=src)
    return P.make_wave_problem(cfg)


def _run(prob, nt, time_block, rec=None, init=None, step0=0):
    op = P.Operator(prob, time_block=time_block, receivers=rec)
    if init is not None:
        for l in range(3):
            op.set_level(l, init[l])
    r = op.apply(nt, step0)
    st = op.stats()
    out = (op.levels(), r.step_max_abs, r.rec_traces, st)
    op.close()
    return out


@pytest.mark.parametrize("so", [2, 4, 8, 12, 16])
@pytest.mark.parametrize("nt", [7, 10])
def test_k3_bitwise_equals_k1(so, nt):
    shape = (46, 40, 75)
    prob = _problem(shape, so, nt)
    rng = np.random.default_rng(so)
    init = [(rng.standard_normal(shape) * 1e-3).astype(np.float32) for _ in range(3)]
    rec = np.array([[x, 20, 37] for x in range(0, shape[0], 3)], np.int32)
    l1, m1, t1, s1 = _run(prob, nt, 1, rec, init)
    l3, m3, t3, s3 = _run(prob, nt, 2, rec, init)
    assert s1.launch_steps == 1 and s3.launch_steps == 2
    assert np.array_equal(l1, l3)
    assert np.array_equal(m1, m3)
    assert np.array_equal(t1, t3)


@pytest.mark.parametrize("cap", [6, 20])
@pytest.mark.parametrize("so", [4, 16])
def test_k3_many_items_per_cta(so, cap, monkeypatch):
    """Few CTAs: every stage-1/stage-2 CTA walks several items (rounds), so stage-2 items
    depend on stage-1 items of later rounds."""
    monkeypatch.setenv("SWB_MAX_CTAS", str(cap))
    shape, nt = (60, 70, 130), 6
    prob = _problem(shape, so, nt, seed=11)
    l1, m1, _, _ = _run(prob, nt, 1)
    l3, m3, _, s3 = _run(prob, nt, 2)
    assert s3.launch_steps == 2
    assert np.array_equal(l1, l3)
    assert np.array_equal(m1, m3)


def test_k3_full_size_256_so8():
    shape, so, nt = (256, 256, 256), 8, 12
    prob = _problem(shape, so, nt, seed=2, damp=0.0)
    l1, m1, _, _ = _run(prob, nt, 1)
    l3, m3, _, s3 = _run(prob, nt, 2)
    assert s3.kernel_launches == nt // 2
    assert np.array_equal(l1, l3)
    assert np.array_equal(m1, m3)


def test_k3_resumable_from_odd_step():
    shape, so = (30, 34, 40), 6
    prob = _problem(shape, so, 20)
    a = P.Operator(prob, time_block=2)
    a.apply(20, 0)
    b = P.Operator(prob, time_block=2)
    b.apply(5, 0)
    b.apply(15)
    c = P.Operator(prob, time_block=1)
    c.apply(20, 0)
    assert np.array_equal(a.levels(), b.levels())
    assert np.array_equal(a.levels(), c.levels())


def test_k3_rejects_deeper_blocking():
    prob = _problem((20, 20, 20), 4, 4)
    with pytest.raises(ValueError):
        P.Operator(prob, time_block=3)


@pytest.mark.parametrize("so", [12, 16])
def test_tmem_queue_variant_bitwise_equals_k1(so, monkeypatch):
    """The K1 variant with the dim-0 queue in tensor memory (SWB_UNR=0; slower, kept
    as an option) runs the same arithmetic, so it must agree with the register queue bit for bit."""
    shape, nt = (52, 54, 70), 9
    prob = _problem(shape, so, nt, seed=so)
    l1, m1, _, s1 = _run(prob, nt, 1)
    monkeypatch.setenv("SWB_UNR", "0")
    monkeypatch.setenv("SWB_T1", "30")
    lt, mt, _, st = _run(prob, nt, 1)
    assert st.kernel_variant % 100 == so // 2 and (st.kernel_variant // 10) % 10 == 0
    assert np.array_equal(l1, lt)
    assert np.array_equal(m1, mt)
