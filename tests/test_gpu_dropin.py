"""The reference tree rebuilt with integration/executor_b200.cpp instead of
src/executor.cpp (integration/_build/dropin_run, built by `make -C integration` where
/root/reference exists): the reference's own call sequence
make_wave_problem -> wave_equations -> lower -> optimize_all -> build_iet -> exec::run
now runs on the B200 kernels.  basic IET: bit-exact with the oracle; aggressive IET:
<= 1e-5 relative L2 (the sign-corrected factorised form)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import bindings as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "integration", "_build", "dropin_run")


def run_dropin(dse, shape, so, steps, damp, tmp_path):
    out = tmp_path / f"{dse}.bin"
    p = subprocess.run([EXE, dse, *map(str, shape), str(so), str(steps), str(damp), str(out)],
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    raw = out.read_bytes()
    fl = int(np.frombuffer(raw[:4], np.int32)[0])
    pu = int(np.frombuffer(raw[4:12], np.uint64)[0])
    smax = np.frombuffer(raw[12:12 + 4 * steps], np.float32)
    levels = np.frombuffer(raw[12 + 4 * steps:], np.float32).reshape((3,) + tuple(shape))
    return fl, pu, smax, levels


@pytest.mark.skipif(not os.path.exists(EXE), reason="drop-in binary not built (needs /root/reference)")
@pytest.mark.parametrize("so,damp", [(2, 0.0), (8, 0.05), (16, 0.0)])
def test_reference_api_runs_on_b200(so, damp, tmp_path):
    shape, steps = (so + 14, so + 15, so + 16), 11
    ref = O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=steps, damp_max=damp, damp_width=4))
    fl, pu, smax, lv = run_dropin("basic", shape, so, steps, damp, tmp_path)
    assert fl == ref["final_level"] and pu == ref["point_updates"]
    assert np.array_equal(lv, ref["levels"]) and np.array_equal(smax, ref["step_max_abs"])
    fl, pu, smax, lv = run_dropin("aggressive", shape, so, steps, damp, tmp_path)
    err = np.linalg.norm(lv[fl] - ref["levels"][fl]) / np.linalg.norm(ref["levels"][fl])
    assert err <= 1e-5


@pytest.mark.skipif(not os.path.exists(EXE), reason="drop-in binary not built (needs /root/reference)")
@pytest.mark.parametrize("dse", ["basic", "aggressive"])
def test_reference_api_instability_error(dse, tmp_path):
    """exec::run on the B200 kernels throws exec::InstabilityError with the first non-finite step,
    as the reference interpreter does (src/executor.cpp:588-593); the basic IET's step equals the
    C restatement's, and the aggressive IET's the Python mirror's factorised run."""
    import paper_1912_00695_b200 as P
    shape, so, steps, dt = (16, 16, 16), 4, 400, 0.02
    p = subprocess.run([EXE, dse, *map(str, shape), str(so), str(steps), "0", str(tmp_path / "x.bin"), str(dt)],
                       capture_output=True, text=True, timeout=120)
    assert p.returncode == 3, p.stdout + p.stderr
    step = int(p.stdout.strip().split("step=")[1])
    if dse == "basic":
        with pytest.raises(O.OracleError) as eo:
            O.port_run(O.OracleConfig(shape=shape, space_order=so, steps=steps, dt=dt))
        assert step == eo.value.step
    else:
        cfg = P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so, steps=steps, dt=dt)
        with pytest.raises(P.InstabilityError) as ei:
            P.run(P.make_wave_problem(cfg), dse=P.DseLevel.aggressive)
        assert step == ei.value.step()


@pytest.mark.skipif(not os.path.exists(EXE), reason="drop-in binary not built (needs /root/reference)")
@pytest.mark.parametrize("dse", ["basic", "aggressive"])
def test_reference_api_on_step_and_check_bounds(dse, tmp_path):
    """RunOptions::on_step through the drop-in: the callback's Field shows the newest level
    (its max|u| is step_max_abs[step]) and the previous newest level unchanged, with one level
    downloaded per step; check_bounds on the canonical tree passes and changes nothing."""
    shape, so, steps = (20, 21, 22), 8, 9
    env = dict(os.environ, DROPIN_ON_STEP="1", DROPIN_CHECK_BOUNDS="1")
    out = tmp_path / "cb.bin"
    p = subprocess.run([EXE, dse, *map(str, shape), str(so), str(steps), "0.05", str(out)],
                       capture_output=True, text=True, timeout=120, env=env)
    assert p.returncode == 0 and "on_step match -1" in p.stdout, p.stdout + p.stderr
    plain = tmp_path / "plain.bin"
    q = subprocess.run([EXE, dse, *map(str, shape), str(so), str(steps), "0.05", str(plain)],
                       capture_output=True, text=True, timeout=120)
    assert q.returncode == 0, q.stdout + q.stderr
    assert out.read_bytes() == plain.read_bytes()
