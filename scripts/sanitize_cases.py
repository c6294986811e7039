"""Small workloads for compute-sanitizer (scripts/sanitize.sh): every kernel family on grids
small enough for the tools' instrumentation -- K1 (TMA 2.5D) at SO 2/4/8/12/16 with damping, the SO 16 y-pencil variant,
source and receivers, the plain FP64/FP32 and factorised one-thread-per-point kernels, z-slabs
with the kernel-ordered exchange and with the fused in-kernel ordering (grid capped so both
persistent grids are co-resident on one GPU), snapshots and the adjoint.
  python scripts/sanitize_cases.py [case ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1912_00695_b200 as P  # noqa: E402


def prob(shape, so, nt, damp=0.05):
    rng = np.random.default_rng(so)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    return P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=damp, damp_width=4))


def k1():
    for so in (2, 4, 8, 12, 16):
        pr = prob((so + 22, so + 26, so + 70), so, 5)
        rec = np.array([[so // 2 + 3, so // 2 + 4, z] for z in range(so // 2, so // 2 + 30, 3)], np.int32)
        P.run(pr, receivers=rec)


def simple():
    for form in ("plain_f64", "plain_f32", "factorised_simple", "factorised_simple_f32c"):
        for so in (4, 8):
            P.run(prob((so + 12, so + 13, so + 14), so, 3), form=form)


def slabs(modes=(False, True)):
    pr = prob((40, 30, 70), 8, 6)
    for fused in modes:
        if fused:
            os.environ["SWB_FUSED_SAME_DEVICE"] = "1"
            os.environ["SWB_MAX_CTAS"] = "40"
        ops = [P.Operator(pr, slab=s) for s in ((0, 14), (14, 27), (27, 40))]
        P.Operator.link_local(ops[0], ops[1])
        P.Operator.link_local(ops[1], ops[2])
        for o in ops:
            o.apply_async(6, 0)
        for o in ops:
            o.collect(6)
        for o in ops:
            o.close()
    os.environ.pop("SWB_FUSED_SAME_DEVICE", None)
    os.environ.pop("SWB_MAX_CTAS", None)


def pencil(fused=True):
    """K1 with the y-pencil warp (SO 16, 20-row tile, forced), single domain and fused slabs."""
    os.environ["SWB_YW"], os.environ["SWB_T1"] = "1", "20"
    pr = prob((40, 50, 70), 16, 5)
    rec = np.array([[20, 25, z] for z in range(8, 60, 5)], np.int32)
    P.run(pr, receivers=rec)
    if fused:
        os.environ["SWB_FUSED_SAME_DEVICE"], os.environ["SWB_MAX_CTAS"] = "1", "60"
        ops = [P.Operator(pr, slab=s) for s in ((0, 20), (20, 40))]
        P.Operator.link_local(ops[0], ops[1])
        for o in ops:
            o.apply_async(5, 0)
        for o in ops:
            o.collect(5)
            o.close()
    for k in ("SWB_YW", "SWB_T1", "SWB_FUSED_SAME_DEVICE", "SWB_MAX_CTAS"):
        os.environ.pop(k, None)


def extras():
    pr = prob((30, 32, 70), 8, 8)
    rec = np.array([[15, 16, z] for z in range(4, 60, 5)], np.int32)
    op = P.Operator(pr, receivers=rec)
    op.apply_snapshots(8, 4, 0)
    op.apply_adjoint(np.ones((8, rec.shape[0]), np.float32))
    op.close()


def slabs_ordered():
    """Kernel-ordered exchange under initcheck.  initcheck serialises the slabs' streams, so a slab
    whose wait kernel spins for a neighbour would block that neighbour (and time out by design); the
    slabs are therefore stepped round-robin, one synchronous step each, which satisfies every wait
    before it is issued.  The fused in-kernel ordering is covered by memcheck/synccheck/racecheck."""
    pr = prob((40, 30, 70), 8, 6)
    ops = [P.Operator(pr, slab=s) for s in ((0, 14), (14, 27), (27, 40))]
    P.Operator.link_local(ops[0], ops[1])
    P.Operator.link_local(ops[1], ops[2])
    for step in range(6):
        for o in ops:
            o.apply(1, step)
    for o in ops:
        o.close()


CASES = {"k1": k1, "pencil": pencil, "pencil_single": lambda: pencil(False), "simple": simple, "slabs": slabs, "slabs_ordered": slabs_ordered, "extras": extras}
if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("case", name, "done", flush=True)
