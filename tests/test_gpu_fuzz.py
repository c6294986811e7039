"""Seeded random configurations against the C restatement: shapes (odd, thin, non-cubic),
every even space order up to 16, damping widths, heterogeneous velocity, source and receivers
anywhere in the interior, random initial levels, step counts that are odd and even.
plain FP64 bit-exact (levels, per-step max, traces); factorised <= 1e-5; K3 == K1 bitwise."""
import os

import numpy as np
import pytest

import paper_1912_00695_b200 as P
from oracle import bindings as O

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    so = int(rng.choice([2, 4, 6, 8, 10, 12, 14, 16]))
    h = so // 2
    shape = tuple(int(rng.integers(2 * h + 3, 2 * h + 40)) for _ in range(3))
    nt = int(rng.integers(3, 30))
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    damp = float(rng.choice([0.0, 0.02, 0.1]))
    width = int(rng.integers(1, 6))
    src = [int(rng.integers(h, s - h)) for s in shape]
    nrec = int(rng.integers(1, 12))
    rec = np.array([[int(rng.integers(0, s)) for s in shape] for _ in range(nrec)], np.int32)
    init = [(rng.standard_normal(shape) * 1e-2).astype(np.float32) for _ in range(3)]
    return so, shape, nt, vel, damp, width, src, rec, init


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SWB_FUZZ_CASES", "64"))))
def test_random_configuration(seed):
    so, shape, nt, vel, damp, width, src, rec, init = _case(seed)
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                              velocity_field=vel, damp_max=damp, damp_width=width, source_point=src)
    prob = P.make_wave_problem(cfg)
    ref = O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=nt, velocity_field=vel, damp_max=damp,
                                    damp_width=width, source_point=src), initial_u=init, receivers=rec)
    opts = P.RunOptions(initial_u=init)
    exact = P.run(prob, opts, dse=P.DseLevel.basic, receivers=rec)
    assert np.array_equal(exact.u.data, ref["levels"])
    assert np.array_equal(exact.step_max_abs, ref["step_max_abs"])
    assert np.array_equal(exact.rec_traces, ref["rec_traces"])
    fast = P.run(prob, opts, dse=P.DseLevel.aggressive, receivers=rec)
    fl = fast.final_level
    assert rel_l2(fast.u.data[fl], ref["levels"][fl]) <= 1e-5
    assert rel_l2(fast.rec_traces, ref["rec_traces"]) <= 1e-5


@pytest.mark.parametrize("seed", range(16))
def test_random_slab_decomposition(seed):
    """Random z-slab cuts (2-4 slabs, each at least SO/2 planes thick) of random problems equal
    the single domain bit for bit, for the factorised and the plain FP64 kernels."""
    so, shape, nt, vel, damp, width, src, rec, init = _case(500 + seed)
    h = so // 2
    rng = np.random.default_rng(77 + seed)
    nslab = int(rng.integers(2, 5))
    cuts = sorted(set(int(c) for c in rng.integers(h, shape[0] - h, size=nslab - 1)))
    bounds = [0] + cuts + [shape[0]]
    if any(b - a < h for a, b in zip(bounds[:-1], bounds[1:])):
        bounds = [0, shape[0] // 2, shape[0]]
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                              velocity_field=vel, damp_max=damp, damp_width=width, source_point=src)
    prob = P.make_wave_problem(cfg)
    for form in ("factorised", "plain_f64"):
        whole = P.Operator(prob, form=form)
        for l in range(3):
            whole.set_level(l, init[l])
        wr = whole.apply(nt, 0)
        ops = [P.Operator(prob, form=form, slab=(bounds[i], bounds[i + 1])) for i in range(len(bounds) - 1)]
        for o in ops:
            for l in range(3):
                o.set_level(l, init[l])
        for lo, hi in zip(ops[:-1], ops[1:]):
            P.Operator.link_local(lo, hi)
        for o in ops:
            o.apply_async(nt, 0)
        smax = np.max([o.collect(nt) for o in ops], axis=0)
        assert np.array_equal(smax, wr.step_max_abs), form
        for l in range(3):
            full = np.zeros(shape, np.float32)
            for o in ops:
                a, b = o.slab
                full[a:b] = o.get_level(l)[a:b]
            assert np.array_equal(full, whole.get_level(l)), (form, l)


@pytest.mark.parametrize("seed", range(24))
def test_random_fused_slab_exchange(seed, monkeypatch):
    """Random z-slab cuts with the fused in-kernel halo ordering (TMA producers wait on the
    neighbours' step counters before loading ghost planes; peer stores of boundary planes; no
    ordering kernels), forced on one GPU with every slab's grid capped so all persistent CTAs
    are co-resident, as they are on separate GPUs.  N slabs == 1 domain bit for bit."""
    so, shape, nt, vel, damp, width, src, rec, init = _case(900 + seed)
    h = so // 2
    rng = np.random.default_rng(313 + seed)
    nslab = int(rng.integers(2, 5))
    cuts = sorted(set(int(c) for c in rng.integers(h, shape[0] - h, size=nslab - 1)))
    bounds = [0] + cuts + [shape[0]]
    if any(b - a < h for a, b in zip(bounds[:-1], bounds[1:])):
        bounds = [0, shape[0] // 2, shape[0]]
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=nt,
                              velocity_field=vel, damp_max=damp, damp_width=width, source_point=src)
    prob = P.make_wave_problem(cfg)
    whole = P.Operator(prob)
    for l in range(3):
        whole.set_level(l, init[l])
    wr = whole.apply(nt, 0)
    monkeypatch.setenv("SWB_FUSED_SAME_DEVICE", "1")
    monkeypatch.setenv("SWB_MAX_CTAS", str(148 // (len(bounds) - 1)))
    ops = [P.Operator(prob, slab=(bounds[i], bounds[i + 1])) for i in range(len(bounds) - 1)]
    for o in ops:
        for l in range(3):
            o.set_level(l, init[l])
    for lo, hi in zip(ops[:-1], ops[1:]):
        P.Operator.link_local(lo, hi)
    for o in ops:
        o.apply_async(nt, 0)
    smax = np.max([o.collect(nt) for o in ops], axis=0)
    # fused ordering: one stencil launch per step and slab, no wait/signal kernels (a slab with
    # no updatable plane has no TMA plan and its sides fall back to ordering kernels)
    if all(max(a, h) < min(b, shape[0] - h) for a, b in zip(bounds[:-1], bounds[1:])):
        assert all(o.stats().kernel_launches == nt for o in ops)
    assert np.array_equal(smax, wr.step_max_abs)
    for l in range(3):
        full = np.zeros(shape, np.float32)
        for o in ops:
            a, b = o.slab
            full[a:b] = o.get_level(l)[a:b]
        assert np.array_equal(full, whole.get_level(l)), l
