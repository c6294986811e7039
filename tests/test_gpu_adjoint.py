"""Adjoint operator on the GPU (swb_apply_adjoint): the transpose of source wavelet ->
receiver traces, run backwards in time with the receivers as injection points.
* plain FP64 kernel: bit-identical to the C restatement (oracle port_adjoint), which is itself
  pinned by the adjoint identity (tests/test_oracle_adjoint.py);
* factorised TMA kernel: relative L2 <= 1e-5 against the restatement;
* the adjoint identity <F w, d> == <w, F^T d> through the product path (forward traces from
  Operator.apply, adjoint from Operator.apply_adjoint)."""
import numpy as np
import pytest

import paper_1912_00695_b200 as P
from oracle import bindings as O

pytestmark = pytest.mark.gpu


def _setup(so, steps=60, shape=(40, 38, 44), seed=0, damp=0.05):
    rng = np.random.default_rng(seed)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    w = rng.standard_normal(steps).astype(np.float32)
    src = [17, 19, 21]
    # receivers: a line through the grid, including points in the never-written ring
    rec = np.array([[x, 12, 30] for x in range(1, shape[0] - 1, 3)], np.int32)
    crec = np.array([[115.5, 203.0, 151.25], [220.0, 133.3, 277.7]], np.float64)
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=steps,
                              velocity_field=vel, damp_max=damp, damp_width=5, source_point=src,
                              source_wavelet=w)
    ocfg = O.OracleConfig(shape=shape, space_order=so, steps=steps, velocity_field=vel, damp_max=damp,
                          damp_width=5, source_point=src, source_wavelet=w)
    return P.make_wave_problem(cfg), ocfg, w, rec, crec, rng


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("so", [2, 4, 8, 16])
def test_plain_f64_adjoint_bit_exact_with_oracle(so):
    prob, ocfg, w, rec, crec, rng = _setup(so)
    d = rng.standard_normal((ocfg.steps, rec.shape[0] + crec.shape[0])).astype(np.float32)
    ref = O.port_adjoint(ocfg, d, receivers=rec, receiver_coords=crec)
    op = P.Operator(prob, form="plain_f64", receivers=rec, receiver_coords=crec)
    got = op.apply_adjoint(d)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("so", [4, 8, 12, 16])
def test_factorised_adjoint_matches_oracle(so):
    prob, ocfg, w, rec, crec, rng = _setup(so, steps=120)
    d = rng.standard_normal((ocfg.steps, rec.shape[0] + crec.shape[0])).astype(np.float32)
    ref = O.port_adjoint(ocfg, d, receivers=rec, receiver_coords=crec)
    op = P.Operator(prob, receivers=rec, receiver_coords=crec)
    got = op.apply_adjoint(d)
    assert rel_l2(got, ref) <= 1e-5


@pytest.mark.parametrize("form", ["factorised", "plain_f64"])
@pytest.mark.parametrize("so", [4, 16])
def test_adjoint_identity_through_the_product_path(form, so):
    prob, ocfg, w, rec, crec, rng = _setup(so, steps=100, seed=so)
    op = P.Operator(prob, form=form, receivers=rec, receiver_coords=crec)
    d = op.apply(ocfg.steps, 0).rec_traces.astype(np.float64)
    dp = rng.standard_normal(d.shape).astype(np.float32)
    wp = op.apply_adjoint(dp).astype(np.float64)
    lhs, rhs = float(np.sum(d * dp)), float(np.sum(w.astype(np.float64) * wp))
    assert abs(lhs - rhs) <= 1e-5 * max(abs(lhs), abs(rhs)), (lhs, rhs)


def test_adjoint_requires_receivers_and_source():
    prob, ocfg, w, rec, crec, rng = _setup(4, steps=10)
    op = P.Operator(prob)
    with pytest.raises(ValueError):
        op.apply_adjoint(np.zeros((10, 0), np.float32))
