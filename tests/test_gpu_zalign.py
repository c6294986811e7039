"""K1's z-tile origin (k_tma.cu tile_z_start): tiles start on a 256-byte boundary at SO <= 12 when
that adds no tile, else at z0 rounded down to a float4.  The origin only changes which lane computes
which point (every point's arithmetic is per point), so both origins must give the same bits: levels,
per-step max|u| and receiver traces, on random damped heterogeneous problems with a source, including
SO 16 forced onto the aligned origin and shapes where alignment would add a tile (then not taken)."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P

pytestmark = pytest.mark.gpu


def _run(monkeypatch, zalign, so, shape, nt, vel, damp, width, src, rec, init):
    monkeypatch.setenv("SWB_ZALIGN", zalign)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp,
                                                   damp_width=width, source_point=src))
    op = P.Operator(prob, receivers=rec)
    for lvl in range(3):
        op.set_level(lvl, init[lvl])
    r = op.apply(nt, 0)
    out = [op.get_level(lvl).copy() for lvl in range(3)], np.array(r.step_max_abs), np.array(r.rec_traces)
    op.close()
    return out


@pytest.mark.parametrize("seed", range(16))
def test_tile_origin_is_bitwise_neutral(seed, monkeypatch):
    rng = np.random.default_rng(5100 + seed)
    so = int(rng.choice([4, 6, 8, 10, 12, 16]))
    h = so // 2
    # n2 spans the cases where the aligned origin keeps the tile count and where it would add one
    shape = (int(rng.integers(2 * h + 3, 2 * h + 40)), int(rng.integers(2 * h + 3, 2 * h + 40)),
             int(rng.integers(2 * h + 3, 2 * h + 150)))
    nt = int(rng.integers(3, 20))
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    damp = float(rng.choice([0.0, 0.05]))
    width = int(rng.integers(1, 5))
    src = [int(rng.integers(h, s - h)) for s in shape]
    rec = np.array([[int(rng.integers(0, s)) for s in shape] for _ in range(4)], np.int32)
    init = [(rng.standard_normal(shape) * 1e-2).astype(np.float32) for _ in range(3)]
    args = (so, shape, nt, vel, damp, width, src, rec, init)
    a_lv, a_mx, a_rc = _run(monkeypatch, "0", *args)
    b_lv, b_mx, b_rc = _run(monkeypatch, "1", *args)
    for lvl in range(3):
        assert np.array_equal(a_lv[lvl], b_lv[lvl]), f"level {lvl} differs (SO {so}, shape {shape})"
    assert np.array_equal(a_mx, b_mx)
    assert np.array_equal(a_rc, b_rc)
