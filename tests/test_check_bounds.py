"""RunOptions::check_bounds (include/stencilc/executor.hpp:74; src/executor.cpp:233, 333, 417-428, 553).

The reference validates every field access of every point against the padded allocation and
throws std::out_of_range("access to <f> leaves the allocation in <dim> at step <s>") at the first
one outside.  The drop-in executor (integration/executor_b200.cpp) finds the same first failing
access without visiting the points; these tests run the same hand-edited trees through the
reference's own interpreter (oracle/_ref/ref_main) and through the drop-in
(integration/_build/dropin_run) and compare the messages.  Everything here fails before any
device work, so it runs on CPU.

Reference defect seen here: the interpreter throws from inside its OpenMP parallel region
(src/executor.cpp:479-482, entered even with one thread), so the exception cannot reach the
caller and the process terminates with the message; the drop-in throws a catchable
std::out_of_range, as executor.hpp documents.
"""
import os
import subprocess

import pytest

import paper_1912_00695_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "ref_main")
DROPIN = os.path.join(ROOT, "integration", "_build", "dropin_run")
need = pytest.mark.skipif(not (os.path.exists(REF) and os.path.exists(DROPIN)),
                          reason="reference checker / drop-in binaries not built (need /root/reference)")


def run(exe, dse, env, shape=(20, 20, 20), so=4, steps=3):
    e = dict(os.environ, DROPIN_CHECK_BOUNDS="1", **env)
    p = subprocess.run([exe, dse, *map(str, shape), str(so), str(steps), "0", "-"], env=e,
                       capture_output=True, text=True, timeout=120)
    return p.returncode, p.stdout + p.stderr


def ref_message(out):
    # terminate called after throwing an instance of 'std::out_of_range'\n  what():  <msg>
    for line in out.splitlines():
        if "what():" in line:
            return line.split("what():", 1)[1].strip()
    return None


# cluster 0 (the stencil) iteration ranges edited to reach past the allocation in each dim, on
# the low and the high side, for u (halo SO/2) and m/damp (halo 1)
CASES = ["0,-3,10", "0,-1,17", "0,2,25", "1,-2,17", "1,2,23", "2,2,22", "0,-4,22", "2,-1,17", "1,0,21"]


@need
@pytest.mark.parametrize("bounds", CASES)
@pytest.mark.parametrize("dse", ["basic", "aggressive"])
def test_first_failing_access_matches_reference(bounds, dse):
    rc_ref, out_ref = run(REF, dse, {"DROPIN_BOUNDS": bounds})
    rc_b2, out_b2 = run(DROPIN, dse, {"DROPIN_BOUNDS": bounds})
    msg = ref_message(out_ref)
    assert msg and msg.startswith("access to "), out_ref
    assert rc_b2 == 4, out_b2
    assert out_b2.strip() == "out_of_range " + msg


@need
@pytest.mark.parametrize("so", [2, 8, 16])
def test_in_bounds_edited_tree_is_rejected_not_run(so):
    """A tree that stays inside the allocation but is not the acoustic operator: the reference
    runs it; the drop-in has no CPU fallback and says so (std::invalid_argument)."""
    h = so // 2
    n = so + 12
    rc_ref, out_ref = run(REF, "basic", {"DROPIN_BOUNDS": f"2,{h},{n - 2 - h}"}, shape=(n, n, n), so=so)
    assert rc_ref == 0 and out_ref.startswith("ok"), out_ref
    rc_b2, out_b2 = run(DROPIN, "basic", {"DROPIN_BOUNDS": f"2,{h},{n - 2 - h}"}, shape=(n, n, n), so=so)
    assert rc_b2 == 1 and "not the acoustic wave operator" in out_b2


def test_mirror_check_bounds_source_outside_allocation():
    """The Python mirror: a source point moved after make_wave_problem.  Outside the padded
    allocation of u (halo SO/2) with check_bounds -> OutOfRangeError with the interpreter's message
    (raised by swb_create before any device work); without check_bounds -> ValueError."""
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=(20, 20, 20), spacing=(10.0, 10.0, 10.0),
                                                   space_order=4, steps=3))
    prob.source.point = [10, -5, 10]
    with pytest.raises(P.OutOfRangeError, match="access to u leaves the allocation in y at step 0"):
        P.run(prob, P.RunOptions(check_bounds=True))
    with pytest.raises(ValueError, match="updatable interior"):
        P.run(prob, P.RunOptions(check_bounds=False))
    prob.source.point = [10, 10, 23]
    with pytest.raises(P.OutOfRangeError, match="in z at step 0"):
        P.run(prob, P.RunOptions(check_bounds=True))
    assert issubclass(P.OutOfRangeError, IndexError)
