"""OPS-text retargeting (second half): the reference's code-generation path
(outline_kernel -> emit_program, /root/reference/proj/src/opsgen.cpp:250-312, 371-614) retargeted to
the B200 operator by integration/opsgen_b200.cpp.  integration/_build/opsgen_b200 runs the
reference's own pipeline, writes the reference's OPS program and the B200 program side by side.

CPU: the emitted program's structure mirrors the OPS host's (one result fetch of u_levels[steps % 3],
the same max|u| line), emission is deterministic, kernels that are not this problem's operator are
rejected, and the host file compiles and links against libswb.so with a plain C compiler.
GPU: the generated program's fetched level equals the Python API's result bit for bit (basic: the
bit-exact kernel, so also the reference's exec::run; aggressive: the factorised kernel)."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GEN = os.path.join(ROOT, "integration", "_build", "opsgen_b200")
LIB = os.path.join(ROOT, "paper_1912_00695_b200", "_lib")
need_gen = pytest.mark.skipif(not os.path.exists(GEN), reason="generator not built (needs /root/reference)")
CC = shutil.which("gcc") or shutil.which("cc")


def generate(tmp_path, dse, shape, so, steps, damp, name="wave", hetero=False, env=None):
    args = [GEN, dse, *map(str, shape), str(so), str(steps), str(damp), str(tmp_path), name]
    if hetero:
        args.append("hetero")
    return subprocess.run(args, capture_output=True, text=True, timeout=120, env=env)


def compile_host(tmp_path, name="wave"):
    exe = tmp_path / f"{name}_host"
    p = subprocess.run([CC, "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
                        str(tmp_path), "-o", str(exe), str(tmp_path / f"{name}_host.c"), "-L", LIB, "-lswb",
                        f"-Wl,-rpath,{LIB}", "-lm"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    return exe


@need_gen
@pytest.mark.parametrize("dse", ["basic", "aggressive"])
def test_generates_b200_program_next_to_ops(tmp_path, dse):
    p = generate(tmp_path, dse, (24, 26, 28), 8, 15, 0.05)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.split()[:2] == ["ok", dse]
    ops = (tmp_path / "ops_wave_host.c").read_text()
    host = (tmp_path / "wave_host.c").read_text()
    kern = (tmp_path / "wave_kernels.h").read_text()
    # the reference's program: one ops_par_loop per kernel per step, fetch of u_levels[15 % 3]
    assert ops.count("ops_par_loop(") == 2 and "ops_dat_fetch_data(u_levels[0]" in ops
    # the B200 program: one swb_apply for the whole loop, the same fetch and output line
    assert host.count("swb_apply(") == 1
    assert not any(t in host for t in ("ops_init(", "ops_par_loop(", "ops_seq.h", "ops_decl_dat("))
    assert "swb_get_level(h, 0, field)" in host
    assert 'printf("max |u| = %g after 15 steps\\n", u_max);' in host and "max |u| = %g after 15 steps" in ops
    form = "SWB_FORM_PLAIN_F64" if dse == "basic" else "SWB_FORM_FACTORISED"
    assert f"#define WAVE_FORM {form}" in kern
    # iteration ranges and stencil points carried over from the OPS stencil declarations
    m = re.search(r"int k0_range\[\] = \{([^}]*)\}", ops)
    assert m and f"wave_k0_range[6] = {{{m.group(1)}}}" in kern
    m = re.search(r"int s3d_k0_ut00_pts\[\] = \{([^}]*)\}", ops)
    assert m and f"wave_k0_ut00_pts[] = {{{m.group(1)}}}" in kern
    # the wavelet travels as exact hex floats
    assert kern.count("p-") + kern.count("p+") >= 15


@need_gen
def test_emission_is_deterministic(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    a.mkdir()
    b.mkdir()
    for d in (a, b):
        assert generate(d, "aggressive", (20, 21, 22), 4, 7, 0.0).returncode == 0
    for f in ("wave_kernels.h", "wave_host.c"):
        assert (a / f).read_bytes() == (b / f).read_bytes()


@need_gen
def test_rejects_kernels_that_are_not_the_operator(tmp_path):
    env = dict(os.environ, OPSGEN_TAMPER="1")
    p = generate(tmp_path, "basic", (20, 21, 22), 4, 7, 0.0, env=env)
    assert p.returncode == 2 and "not the acoustic wave operator" in p.stdout
    p = generate(tmp_path, "aggressive", (20, 21, 22), 4, 7, 0.0, name="9bad")
    assert p.returncode == 2 and "C identifier" in p.stdout


@need_gen
@pytest.mark.skipif(CC is None, reason="no C compiler")
@pytest.mark.parametrize("hetero", [False, True])
def test_host_program_compiles_against_libswb(tmp_path, hetero):
    assert generate(tmp_path, "aggressive", (24, 26, 28), 8, 9, 0.05, hetero=hetero).returncode == 0
    exe = compile_host(tmp_path)
    assert exe.exists()
    if hetero:
        assert (tmp_path / "wave_m.f32").stat().st_size == 24 * 26 * 28 * 4


@pytest.mark.gpu
@need_gen
@pytest.mark.skipif(CC is None, reason="no C compiler")
@pytest.mark.parametrize("dse,so,damp,hetero", [("basic", 2, 0.0, False), ("basic", 8, 0.05, True),
                                                ("aggressive", 8, 0.05, False), ("aggressive", 16, 0.0, True)])
def test_generated_program_matches_api_bitwise(tmp_path, dse, so, damp, hetero):
    import paper_1912_00695_b200 as P
    shape, steps = (so + 20, so + 22, so + 24), 13
    assert generate(tmp_path, dse, shape, so, steps, damp, hetero=hetero).returncode == 0
    exe = compile_host(tmp_path)
    res_path = tmp_path / "result.f32"
    p = subprocess.run([str(exe), "0", str(res_path)], capture_output=True, text=True, timeout=120,
                       cwd=str(tmp_path))
    assert p.returncode == 0, p.stdout + p.stderr
    got = np.fromfile(res_path, np.float32).reshape(shape)
    vel = np.fromfile(tmp_path / "wave_velocity.f32", np.float32).reshape(shape) if hetero else None
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=steps, velocity_field=vel, damp_max=damp,
                                                   damp_width=4))
    ref = P.run(prob, dse=P.DseLevel[dse])
    want = ref.u.data[steps % 3]
    assert np.array_equal(got, want)
    umax = float(p.stdout.split("=")[1].split()[0])
    assert umax == pytest.approx(float(np.max(np.abs(want))), rel=1e-5)
