"""Pin the CPU oracle (oracle/port, the C restatement) before trusting it:
  * against the golden fixtures generated from the reference itself (tests/golden/),
  * against the reference's own build (oracle/_ref) on fresh random problems when present,
  * against the SPEC.md known-answer examples and an independent Taylor-table solve."""
import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import bindings as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
CASES = [k for k in META if k != "kat"]


def load_case(name):
    m = META[name]
    z = np.load(os.path.join(GOLD, name + ".npz"))
    vel = z["velocity"] if "velocity" in z else None
    init = list(z["initial_u"]) if "initial_u" in z else None
    cfg = O.OracleConfig(shape=tuple(m["shape"]), space_order=m["space_order"], steps=m["steps"],
                         velocity_field=vel, damp_max=m["damp_max"], damp_width=m["damp_width"])
    return m, z, cfg, init


@pytest.mark.parametrize("name", CASES)
def test_port_matches_reference_goldens(name):
    m, z, cfg, init = load_case(name)
    out = O.port_run(cfg, initial_u=init, receivers=z["receivers"])
    for l in range(3):
        assert hashlib.sha256(out["levels"][l].tobytes()).hexdigest() == m["levels_sha256"][l]
    if "levels" in z:
        assert np.array_equal(out["levels"], z["levels"])
    assert np.array_equal(out["step_max_abs"], z["step_max_abs"])
    assert np.array_equal(out["rec_traces"], z["rec_traces"])
    assert out["point_updates"] == m["point_updates"]
    assert out["final_level"] == m["final_level"]
    info = O.port_info(cfg)
    assert np.float32(info["dt"]) == z["dt"]
    assert np.array_equal(info["wavelet"], z["wavelet"])
    assert list(info["source_point"]) == m["source_point"]
    assert [list(w) for w in info["weights"]] == m["weights"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("so", [2, 4, 6, 8, 10, 12, 14, 16])
def test_port_bit_identical_to_reference_build(so):
    rng = np.random.default_rng(so)
    shape = (so + 6 + so % 3, so + 7, so + 5)
    vel = (1500 + 1500 * rng.random(shape)).astype(np.float32)
    init = [(rng.standard_normal(shape) * 1e-3).astype(np.float32) for _ in range(3)]
    cfg = O.OracleConfig(shape=shape, space_order=so, steps=5, velocity_field=vel, damp_max=0.03,
                         damp_width=2, source_point=[shape[0] // 2 - 1, so // 2, shape[2] - 1 - so // 2])
    rec = [[shape[0] // 2, shape[1] // 2, z] for z in range(shape[2])]
    a = O.ref_run(cfg, initial_u=init, receivers=rec)
    b = O.port_run(cfg, initial_u=init, receivers=rec)
    assert np.array_equal(a["levels"], b["levels"])
    assert np.array_equal(a["step_max_abs"], b["step_max_abs"])
    assert np.array_equal(a["rec_traces"], b["rec_traces"])
    assert a["point_updates"] == b["point_updates"]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_run_equals_serial_tree_walker():
    """exec::run == exec::reference_run (include/stencilc/executor.hpp:93-96)."""
    cfg = O.OracleConfig(shape=(12, 12, 12), space_order=4, steps=4, damp_max=0.1, damp_width=3)
    a = O.ref_run(cfg, threads=4)
    b = O.ref_run(cfg, serial=True)
    assert np.array_equal(a["levels"], b["levels"])


def taylor_weights(d, p):
    """Independent exact Gaussian elimination of the Taylor system (src/fd_coefficients.cpp:5-14)."""
    half, n = p // 2, p + 1
    import math
    m = [[Fraction((j - half) ** k) for j in range(n)] + [Fraction(math.factorial(k) if k == d else 0)]
         for k in range(n)]
    for c in range(n):
        piv = next(r for r in range(c, n) if m[r][c] != 0)
        m[c], m[piv] = m[piv], m[c]
        inv = 1 / m[c][c]
        m[c] = [v * inv for v in m[c]]
        for r in range(n):
            if r != c and m[r][c] != 0:
                f = m[r][c]
                m[r] = [a - f * b for a, b in zip(m[r], m[c])]
    return [m[j][n] for j in range(n)]


@pytest.mark.parametrize("p", list(range(2, 25, 2)))
def test_weights_equal_taylor_solve(p):
    import ctypes as C
    lib = O._lib("port")
    num, den = (C.c_int64 * (p + 1))(), (C.c_int64 * (p + 1))()
    assert lib.port_fd_weights(p, num, den) == 0
    got = [Fraction(num[i], den[i]) for i in range(p + 1)]
    assert got == taylor_weights(2, p)


def test_spec_known_answers():
    kat = META["kat"]
    # SPEC.md:58-60 fd_coefficients examples
    assert [Fraction(a, b) for a, b in kat["2"]["weights"]] == [1, -2, 1]
    assert [Fraction(a, b) for a, b in kat["4"]["weights"]] == [Fraction(-1, 12), Fraction(4, 3),
                                                                 Fraction(-5, 2), Fraction(4, 3),
                                                                 Fraction(-1, 12)]
    # SO 8 weights, flop counts of both forms
    assert [Fraction(a, b) for a, b in kat["8"]["weights"]][4:] == [Fraction(-205, 72), Fraction(8, 5),
                                                                     Fraction(-1, 5), Fraction(8, 315),
                                                                     Fraction(-1, 560)]
    assert [kat[s]["flops_basic"] for s in ("2", "4", "8", "12", "16")] == [69, 105, 165, 225, 285]
    assert [kat[s]["flops_aggressive"] for s in ("2", "4", "8", "12", "16")] == [24, 34, 57, 75, 93]
    # SPEC.md:256 256^3 SO 8 source at the centre
    assert kat["8"]["source_point"] == [128, 128, 128]


def test_ricker_known_answers():
    lib = O._lib("port")
    import ctypes as C
    lib.port_ricker_amplitude.restype = C.c_double
    lib.port_ricker_amplitude.argtypes = [C.c_double, C.c_double]
    assert lib.port_ricker_amplitude(10.0, 0.0) == 1.0
    t0 = 1.0 / (np.pi * 10.0 * np.sqrt(2.0))  # SPEC.md:321 zero crossing
    assert abs(lib.port_ricker_amplitude(10.0, t0)) < 1e-12
