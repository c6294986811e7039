"""CPU-side checks of the drop-in boundary: libswb.so loads and exports every symbol that
include/swb.h declares; the host-side model helpers reproduce the reference's problem
setup bit-for-bit; validation errors mirror the reference's messages."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1912_00695_b200 as P
from paper_1912_00695_b200 import _native as N
from oracle import bindings as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "swb.h")).read()
    return sorted(set(re.findall(r"\b(swb_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 19
    lib = C.CDLL(N.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(N.EXPORTED) == syms


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {N.LIB_PATH} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("so,damp", [(2, 0.0), (8, 0.05), (16, 0.2)])
def test_model_helpers_match_port(so, damp):
    shape = (20, 24, 22)
    rng = np.random.default_rng(so)
    vel = (1400 + 1600 * rng.random(shape)).astype(np.float32)
    cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 12.5, 7.5), space_order=so, steps=37,
                              velocity_field=vel, damp_max=damp, damp_width=5)
    prob = P.make_wave_problem(cfg)
    info = O.port_info(O.OracleConfig(shape=shape, spacing=(10.0, 12.5, 7.5), space_order=so,
                                      steps=37, velocity_field=vel, damp_max=damp, damp_width=5))
    assert np.float32(prob.dt) == np.float32(info["dt"])
    assert np.array_equal(prob.source.wavelet, info["wavelet"])
    assert np.array_equal(prob.m_data(), info["m"])
    assert np.array_equal(prob.damp_data(), info["damp"])
    assert list(prob.source.point) == list(info["source_point"])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_model_helpers_match_reference_build():
    cfg = O.OracleConfig(shape=(30, 31, 32), space_order=12, steps=50, damp_max=0.3, damp_width=7)
    info = O.ref_info(cfg)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(30, 31, 32), spacing=(10, 10, 10),
                                                   space_order=12, steps=50, damp_max=0.3,
                                                   damp_width=7))
    assert np.float32(prob.dt) == np.float32(info["dt"])
    assert np.array_equal(prob.source.wavelet, info["wavelet"])
    assert np.array_equal(prob.damp_data(), info["damp"])
    w = [(f.numerator, f.denominator) for _, f in P.fd_coefficients(2, 12)]
    assert w == [tuple(x) for x in info["weights"]]


def test_spec_cfl_examples():
    # 1-D c=1 h=1 so=2 -> 0.9; 3-D -> 0.9/sqrt(3); doubling c halves dt
    one = (C.c_double * 3)(1.0, 1.0, 1.0)
    assert abs(N.lib.swb_cfl_dt(1, one, 1.0, 2) - 0.9) < 1e-15
    assert abs(N.lib.swb_cfl_dt(3, one, 1.0, 2) - 0.9 / np.sqrt(3)) < 1e-15
    assert abs(N.lib.swb_cfl_dt(3, one, 2.0, 8) * 2 - N.lib.swb_cfl_dt(3, one, 1.0, 8)) < 1e-15


@pytest.mark.parametrize("kw,msg", [
    (dict(space_order=3), "space_order must be an even integer >= 2"),
    (dict(time_order=1), "time_order must be 2"),
    (dict(steps=0), "steps must be >= 1"),
    (dict(velocity=-1.0), "velocity must be positive"),
    (dict(source_point=[1, 8, 8]), "source point must lie in the updatable interior"),
    (dict(damp_max=-1.0), "damp_max must be nonnegative"),
])
def test_validation_messages(kw, msg):
    base = dict(shape=(16, 16, 16), spacing=(10, 10, 10), space_order=4, steps=5)
    base.update(kw)
    with pytest.raises(ValueError, match=msg):
        P.make_wave_problem(P.WaveProblemConfig(**base))


def test_no_cpu_fallback_without_gpu():
    """The product path must fail loudly when no B200 is present."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(12, 12, 12), spacing=(10, 10, 10),
                                                   space_order=2, steps=2))
    with pytest.raises(N.CudaError):
        P.run(prob)


def test_write_snapshot_format(tmp_path):
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(4, 5, 6), spacing=(10, 12.5, 7), space_order=2,
                                                   steps=2))
    f = P.Field(prob, np.arange(3 * 120, dtype=np.float32).reshape(3, 4, 5, 6))
    base = P.write_snapshot(str(tmp_path), "u", 7, f, 1, prob)
    assert base.endswith("u_000007")
    data = np.fromfile(base + ".f32", "<f4")
    assert np.array_equal(data, np.arange(120, 240, dtype=np.float32))
    assert open(base + ".meta").read() == "shape=4,5,6\nspacing=10,12.5,7\nstep=7\n"


def test_snapshot_round_trip(tmp_path):
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(5, 6, 7), spacing=(10.0, 12.5, 15.0), space_order=2, steps=3))
    rng = np.random.default_rng(0)
    lev = rng.standard_normal((3, 5, 6, 7)).astype(np.float32)
    base = P.write_snapshot(str(tmp_path), "u", 12, P.Field(prob, lev), 2, prob)
    data, meta = P.read_snapshot(base)
    assert np.array_equal(data, lev[2])
    assert meta == {"shape": (5, 6, 7), "spacing": (10.0, 12.5, 15.0), "step": 12}


def _raw_problem(shape=(16, 16, 16), so=4, **kw):
    p = N.SwbProblem()
    for d in range(3):
        p.shape[d] = shape[d]
        p.spacing[d] = 10.0
    p.space_order = so
    p.dt = 0.001
    m = np.full(shape, 1.0 / 1500.0 ** 2, np.float32)
    p.m = N.fptr(m)
    p.form = 0
    p.time_block = 1
    for k, v in kw.items():
        setattr(p, k, N.fptr(None) if v is None else v)
    return p, m


@pytest.mark.parametrize("kw,msg", [
    (dict(so=5), "space_order must be an even integer"),
    (dict(so=26), "space_order above 24"),
    (dict(shape=(8, 16, 16), so=8), "too small for halo"),
    (dict(time_block=3), "time_block must be 1"),
    (dict(time_block=2), "is retired"),
    (dict(m=None), "or the velocity is required"),
    (dict(form=9), "unknown stencil form"),
    (dict(dt=0.0), "dt must be positive"),
    (dict(slab_lo=0, slab_hi=3, so=8), "slab thinner than SO/2 planes"),
    (dict(slab_lo=10, slab_hi=5), "bad slab range"),
    (dict(n_receivers=2), "bad receiver list"),
])
def test_capi_validation_before_device(kw, msg):
    """swb_create validates the problem (the reference's std::invalid_argument cases) before it
    touches a device, so these paths are exercised here without a GPU."""
    so = kw.pop("so", 4)
    shape = kw.pop("shape", (16, 16, 16))
    p, keep = _raw_problem(shape, so, **kw)
    h = C.c_void_p()
    rc = N.lib.swb_create(C.byref(p), C.byref(h))
    assert rc == N.SWB_EINVAL
    assert msg in N.last_error()


def test_capi_null_arguments():
    h = C.c_void_p()
    assert N.lib.swb_create(None, C.byref(h)) == N.SWB_EINVAL
    assert N.lib.swb_destroy(None) == N.SWB_OK
    assert N.lib.swb_apply(None, 0, 1, None, None, None) == N.SWB_EINVAL
    assert N.lib.swb_apply_adjoint(None, 1, None, None, None, None) == N.SWB_EINVAL
