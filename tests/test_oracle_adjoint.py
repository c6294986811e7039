"""The oracle's adjoint restatement (oracle/port/wave_port.c port_adjoint) is pinned by the
adjoint identity against the forward restatement -- itself pinned bit-for-bit to the
reference's exec::run (test_oracle.py): <F w, d> == <w, F^T d> for random w, d."""
import numpy as np
import pytest

from oracle import bindings as O


def _case(so, damp, seed, steps=40, shape=(34, 34, 36)):
    rng = np.random.default_rng(seed)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    w = rng.standard_normal(steps).astype(np.float32)
    cfg = O.OracleConfig(shape=shape, space_order=so, steps=steps, velocity_field=vel, damp_max=damp,
                         damp_width=4, source_point=[11, 9, 12], source_wavelet=w)
    rec = np.array([[x, 10, 7] for x in range(2, shape[0] - 2, 3)] + [[11, 9, 12]], np.int32)
    crec = np.array([[55.5, 93.0, 101.25], [120.0, 33.3, 77.7]], np.float64)
    return cfg, w, rec, crec, rng


@pytest.mark.parametrize("so,damp", [(2, 0.0), (4, 0.05), (8, 0.05), (16, 0.05)])
def test_port_adjoint_dot_product(so, damp):
    cfg, w, rec, crec, rng = _case(so, damp, seed=so)
    fwd = O.port_run(cfg, receivers=rec, receiver_coords=crec)
    d = np.concatenate([fwd["rec_traces"], fwd["coord_traces"]], axis=1).astype(np.float64)
    dp = rng.standard_normal(d.shape).astype(np.float32)
    wp = O.port_adjoint(cfg, dp, receivers=rec, receiver_coords=crec).astype(np.float64)
    lhs = float(np.sum(d * dp))
    rhs = float(np.sum(w.astype(np.float64) * wp))
    # receivers in the never-written ring (x = 2, 5 at SO 8/16; z = 7 at SO 16) are included
    # on purpose: their adjoint must vanish
    assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), abs(rhs)), (lhs, rhs)


def test_port_adjoint_is_linear():
    cfg, w, rec, crec, rng = _case(4, 0.05, seed=3, steps=25)
    d1 = rng.standard_normal((25, rec.shape[0] + 2)).astype(np.float32)
    d2 = rng.standard_normal((25, rec.shape[0] + 2)).astype(np.float32)
    a1 = O.port_adjoint(cfg, d1, receivers=rec, receiver_coords=crec).astype(np.float64)
    a2 = O.port_adjoint(cfg, d2, receivers=rec, receiver_coords=crec).astype(np.float64)
    a12 = O.port_adjoint(cfg, d1 + 2 * d2, receivers=rec, receiver_coords=crec).astype(np.float64)
    assert np.linalg.norm(a12 - (a1 + 2 * a2)) <= 1e-5 * np.linalg.norm(a12)
