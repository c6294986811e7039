"""K1 with the y-pencil warp (the SO 16 20-row variant: one warp computes the far y terms
k >= 4 of every output plane into a shared-memory ring, k_tma.cu ypencil_loop), forced with
SWB_YW=1 / SWB_T1=20 on every configuration the plain K1 is tested on: random problems against
the C restatement of the reference (<= 1e-5), fused z-slab exchange bitwise equal to one domain,
10k steps within 1e-5, and the plan's choice (pencil at 256^3 and 512^3 SO 16, the 22-row tile
without it at 320^3, where 22-row columns fill the SMs better)."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P
from oracle import bindings as O

pytestmark = pytest.mark.gpu


def pencil_variant(op):
    """kernel_variant = 1000 + 100 (R1 - 1) + 10 UNR + H + 100000 T1 + 10000000 YW (tma_plan)."""
    v = op.stats().kernel_variant
    return v // 10000000, (v // 100000) % 100


@pytest.fixture
def force_pencil(monkeypatch):
    monkeypatch.setenv("SWB_YW", "1")
    monkeypatch.setenv("SWB_T1", "20")


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def _case(seed):
    rng = np.random.default_rng(4000 + seed)
    so, h = 16, 8
    shape = tuple(int(rng.integers(2 * h + 3, 2 * h + 48)) for _ in range(3))
    nt = int(rng.integers(3, 25))
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    damp = float(rng.choice([0.0, 0.02, 0.1]))
    width = int(rng.integers(1, 6))
    src = [int(rng.integers(h, s - h)) for s in shape]
    rec = np.array([[int(rng.integers(0, s)) for s in shape] for _ in range(6)], np.int32)
    init = [(rng.standard_normal(shape) * 1e-2).astype(np.float32) for _ in range(3)]
    return so, shape, nt, vel, damp, width, src, rec, init


@pytest.mark.parametrize("seed", range(12))
def test_pencil_random_configuration(seed, force_pencil):
    so, shape, nt, vel, damp, width, src, rec, init = _case(seed)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp,
                                                   damp_width=width, source_point=src))
    ref = O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=nt, velocity_field=vel, damp_max=damp,
                                    damp_width=width, source_point=src), initial_u=init, receivers=rec)
    op = P.Operator(prob, receivers=rec)
    assert pencil_variant(op) == (1, 20)
    for l in range(3):
        op.set_level(l, init[l])
    r = op.apply(nt, 0)
    fl = nt % 3
    assert rel_l2(op.get_level(fl), ref["levels"][fl]) <= 1e-5
    assert rel_l2(r.rec_traces, ref["rec_traces"]) <= 1e-5


def test_pencil_equals_plain_k1_to_rounding(force_pencil, monkeypatch):
    """The pencil changes only the summation order of the far y terms: the two K1 variants agree
    to FP32 rounding after 50 steps on a damped heterogeneous 96^3 problem."""
    shape, nt = (96, 100, 104), 50
    rng = np.random.default_rng(3)
    vel = (1500.0 + 1500.0 * rng.random(shape)).astype(np.float32)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10., 10., 10.), space_order=16, steps=nt,
                                                   velocity_field=vel, damp_max=0.05, damp_width=6))
    a = P.Operator(prob)
    assert pencil_variant(a) == (1, 20)
    a.apply(nt, 0)
    monkeypatch.setenv("SWB_YW", "0")
    b = P.Operator(prob)
    assert pencil_variant(b) == (0, 20)
    b.apply(nt, 0)
    assert rel_l2(a.get_level(nt % 3), b.get_level(nt % 3)) <= 1e-6


@pytest.mark.parametrize("seed", range(6))
def test_pencil_fused_slab_exchange_bitwise(seed, force_pencil, monkeypatch):
    """Random z-slab cuts with the in-kernel halo ordering (co-resident capped grids on one GPU):
    N slabs == 1 domain bit for bit with the pencil variant on every slab."""
    so, shape, nt, vel, damp, width, src, rec, init = _case(700 + seed)
    h = so // 2
    rng = np.random.default_rng(55 + seed)
    nslab = int(rng.integers(2, 4))
    cuts = sorted(set(int(c) for c in rng.integers(h, shape[0] - h, size=nslab - 1)))
    bounds = [0] + cuts + [shape[0]]
    if any(b - a < h for a, b in zip(bounds[:-1], bounds[1:])):
        bounds = [0, shape[0] // 2, shape[0]]
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp,
                                                   damp_width=width, source_point=src))
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
    assert np.array_equal(smax, wr.step_max_abs)
    for l in range(3):
        full = np.zeros(shape, np.float32)
        for o in ops:
            a, b = o.slab
            full[a:b] = o.get_level(l)[a:b]
        assert np.array_equal(full, whole.get_level(l)), l


def test_pencil_10k_steps_128(force_pencil):
    n, nt = 128, 10000
    shape = (n, n, n)
    rng = np.random.default_rng(16)
    prob = P.make_wave_problem(P.WaveProblemConfig(
        shape=shape, spacing=(10.0, 10.0, 10.0), space_order=16, steps=nt,
        velocity_field=(1500 + 1500 * rng.random(shape)).astype(np.float32), damp_max=0.05, damp_width=10))
    exact = P.Operator(prob, form="plain_f64")
    fast = P.Operator(prob)
    assert pencil_variant(fast) == (1, 20)
    exact.apply(nt, 0)
    fast.apply(nt, 0)
    assert rel_l2(fast.get_level(nt % 3), exact.get_level(nt % 3)) <= 1e-5


@pytest.mark.parametrize("n,so,expect", [(256, 16, (1, 20)), (512, 16, (1, 20)), (320, 16, (0, 22)),
                                           (256, 12, (1, 28)), (512, 12, (1, 28))])
def test_plan_picks_pencil_where_faster(n, so, expect):
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(n,) * 3, spacing=(10., 10., 10.), space_order=so,
                                                   steps=1))
    op = P.Operator(prob)
    assert pencil_variant(op) == expect
    op.close()


@pytest.mark.parametrize("seed", range(12))
def test_pencil_so12_random_configuration(seed, monkeypatch):
    """The SO 12 pencil variant (28-row tile, pencil rows in two sub-segments, P_y through the aux
    ring) forced on random damped heterogeneous problems against the C restatement (<= 1e-5)."""
    monkeypatch.setenv("SWB_YW", "1")
    monkeypatch.setenv("SWB_T1", "28")
    rng = np.random.default_rng(6100 + seed)
    so, h = 12, 6
    shape = tuple(int(rng.integers(2 * h + 3, 2 * h + 60)) for _ in range(3))
    nt = int(rng.integers(3, 25))
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    damp = float(rng.choice([0.0, 0.02, 0.1]))
    width = int(rng.integers(1, 6))
    src = [int(rng.integers(h, s - h)) for s in shape]
    rec = np.array([[int(rng.integers(0, s)) for s in shape] for _ in range(6)], np.int32)
    init = [(rng.standard_normal(shape) * 1e-2).astype(np.float32) for _ in range(3)]
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp,
                                                   damp_width=width, source_point=src))
    ref = O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=nt, velocity_field=vel, damp_max=damp,
                                    damp_width=width, source_point=src), initial_u=init, receivers=rec)
    op = P.Operator(prob, receivers=rec)
    assert pencil_variant(op) == (1, 28)
    for lvl in range(3):
        op.set_level(lvl, init[lvl])
    r = op.apply(nt, 0)
    fl = nt % 3
    assert rel_l2(op.get_level(fl), ref["levels"][fl]) <= 1e-5
    assert rel_l2(r.rec_traces, ref["rec_traces"]) <= 1e-5
