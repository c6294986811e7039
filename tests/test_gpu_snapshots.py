"""Wavefield snapshots overlapped with stepping (swb_apply_snapshots): every snapshot equals
the newest level of a plain stepped run at that step, bit for bit, and the per-step outputs
equal swb_apply's.  Covers K1 (several intervals) and the plain form."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P

pytestmark = pytest.mark.gpu


def _prob(so=8, nt=24, shape=(36, 40, 70)):
    rng = np.random.default_rng(4)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    return P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=0.05, damp_width=4))


@pytest.mark.parametrize("form,every", [("factorised", 5), ("factorised", 1), ("factorised", 4),
                                        ("factorised", 3), ("plain_f64", 6)])
def test_snapshots_equal_stepped_levels(form, every):
    nt = 24
    prob = _prob(nt=nt)
    rec = np.array([[18, 20, z] for z in range(5, 65, 7)], np.int32)
    ref = P.Operator(prob, form=form, receivers=rec)
    want, smax_ref, tr_ref = [], [], []
    for s in range(nt):
        r = ref.apply(1, s)
        smax_ref.append(r.step_max_abs[0])
        tr_ref.append(r.rec_traces[0])
        if (s + 1) % every == 0:
            want.append(ref.get_level((s + 1) % 3))
    op = P.Operator(prob, form=form, receivers=rec)
    res, snaps = op.apply_snapshots(nt, every, 0)
    assert len(snaps) == nt // every
    for i, (a, b) in enumerate(zip(snaps, want)):
        assert np.array_equal(a, b), i
    assert np.array_equal(res.step_max_abs, np.array(smax_ref, np.float32))
    assert np.array_equal(res.rec_traces, np.array(tr_ref))
    assert np.array_equal(op.levels(), ref.levels())


def test_snapshots_validate_buffer_count():
    prob = _prob(nt=10)
    op = P.Operator(prob)
    with pytest.raises(ValueError):
        op.apply_snapshots(10, 3, 0, out=[np.zeros(prob.shape, np.float32)])


@pytest.mark.parametrize("form", ["factorised", "plain_f64"])
def test_checkpoint_restart_bitwise(form, tmp_path):
    """write_checkpoint + Operator.restore (reference snapshot format, two levels) resumes a run
    exactly: 11 + 13 steps through a checkpoint == 24 steps straight."""
    prob = _prob(nt=24)
    rec = np.array([[18, 20, z] for z in range(5, 65, 9)], np.int32)
    straight = P.Operator(prob, form=form, receivers=rec)
    rs = straight.apply(24, 0)
    first = P.Operator(prob, form=form, receivers=rec)
    first.apply(11, 0)
    P.write_checkpoint(str(tmp_path), "ck", first)
    second = P.Operator(prob, form=form, receivers=rec)
    second.restore(str(tmp_path), "ck", 11)
    r2 = second.apply(13)
    nl = 24 % 3
    assert np.array_equal(second.get_level(nl), straight.get_level(nl))
    assert np.array_equal(second.get_level((24 + 2) % 3), straight.get_level((24 + 2) % 3))
    assert np.array_equal(r2.rec_traces, rs.rec_traces[11:])


def test_snapshots_on_linked_slabs():
    """Each slab drains its own planes into the grid-sized snapshot buffers; together they equal
    the single-domain snapshots."""
    nt, every = 12, 4
    prob = _prob(nt=nt)
    whole = P.Operator(prob)
    _, ref = whole.apply_snapshots(nt, every, 0)
    bounds = [0, 13, 24, prob.shape[0]]
    ops = [P.Operator(prob, slab=(bounds[i], bounds[i + 1])) for i in range(3)]
    for lo, hi in zip(ops[:-1], ops[1:]):
        P.Operator.link_local(lo, hi)
    import threading
    import torch
    # pinned buffers: a pageable D2H can block its host thread inside the driver while the other
    # slabs' threads still have to enqueue the steps it depends on
    snaps = [torch.zeros(prob.shape, dtype=torch.float32, pin_memory=True).numpy() for _ in range(nt // every)]
    errs = []

    def run(o):
        try:
            o.apply_snapshots(nt, every, 0, out=snaps)
        except Exception as e:  # pragma: no cover
            errs.append(e)
    th = [threading.Thread(target=run, args=(o,)) for o in ops]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    for a, b in zip(snaps, ref):
        assert np.array_equal(a, b)


def test_adjoint_rejects_linked_slabs():
    prob = _prob(nt=6)
    rec = np.array([[18, 20, 30]], np.int32)
    a = P.Operator(prob, receivers=rec, slab=(0, 18))
    b = P.Operator(prob, receivers=rec, slab=(18, prob.shape[0]))
    P.Operator.link_local(a, b)
    with pytest.raises(ValueError):
        a.apply_adjoint(np.zeros((6, 1), np.float32))
