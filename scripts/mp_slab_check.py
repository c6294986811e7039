"""Multi-process z-slab check (launched by torchrun; ranks may share one GPU).
Each rank owns a slab, links its ghost planes to its neighbours through CUDA IPC, and runs
nt steps; rank 0 compares the gathered levels bit-for-bit with a single-domain run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1912_00695_b200 as P  # noqa: E402
from paper_1912_00695_b200 import dist as D  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    device = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    form = sys.argv[1] if len(sys.argv) > 1 else "factorised"
    so = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    shape, nt = ((40, 24, 26) if so <= 8 else (60, 30, 40)), 17
    rng = np.random.default_rng(11)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=0.05, damp_width=4,
                                                   source_point=[15, 12, 13]))
    rec = np.array([[x, 12, 13] for x in range(shape[0])], np.int32)  # (on-grid line through the slabs)
    slab = D.slab_bounds(shape[0], world, rank)
    op = P.Operator(prob, form=form, device=device, slab=slab, receivers=rec)
    D.exchange_and_link(op, rank, world)
    r = op.apply(nt, 0)
    smax = D.reduce_step_max(r.step_max_abs)
    traces = D.reduce_traces(r.rec_traces)
    levels = [D.gather_level(op.get_level(l), slab) for l in range(3)]
    if rank == 0:
        ref = P.Operator(prob, form=form, device=device, receivers=rec)
        rr = ref.apply(nt, 0)
        ok = all(np.array_equal(levels[l], ref.get_level(l)) for l in range(3))
        ok &= np.array_equal(smax, rr.step_max_abs)
        ok &= np.array_equal(traces, rr.rec_traces)
        print("MP_SLAB_OK" if ok else "MP_SLAB_MISMATCH", world, form, flush=True)
    dist.barrier()
    op.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
