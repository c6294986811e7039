"""Z-slabs on two physical devices (skipped when fewer than two GPUs are visible; the round-end
tiers here have one GPU, the driver's scaling runs have eight).

* two handles of one process on devices 0 and 1, linked with swb_link_local: the halo exchange is
  ordered inside the stencil kernel (fused) over peer memory -- one launch per step -- and the
  result equals one domain bit for bit;
* bench.py --gpus 2 (self-launched under torch.distributed.run): both ranks report a fused link to
  the other device, n_gpus = 2.
The one-GPU tests (test_gpu_multiproc.py, test_gpu_fuzz.py, test_gpu_parity.py) cover the same
code paths with slabs sharing a device."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1912_00695_b200 as P

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count()


needs2 = pytest.mark.skipif(ngpus() < 2, reason="needs two GPUs")


@needs2
@pytest.mark.parametrize("so", [4, 8, 16])
def test_two_device_slabs_bitwise(so):
    shape, nt = (96, 70, 72), 23
    rng = np.random.default_rng(so)
    vel = (1500 + 1000 * rng.random(shape)).astype(np.float32)
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt, velocity_field=vel, damp_max=0.05, damp_width=6,
                                                   source_point=[45, 33, 36]))
    init = [(1e-3 * rng.standard_normal(shape)).astype(np.float32) for _ in range(3)]
    one = P.Operator(prob)
    for l in range(3):
        one.set_level(l, init[l])
    r1 = one.apply(nt, 0)
    ref = one.levels()
    one.close()
    a = P.Operator(prob, device=0, slab=(0, 50))
    b = P.Operator(prob, device=1, slab=(50, 96))
    P.Operator.link_local(a, b)
    sa, sb = a.stats(), b.stats()
    assert sa.fused_hi == 1 and sb.fused_lo == 1, "cross-device slabs must use the in-kernel ordering"
    assert sa.peer_hi == 1 and sb.peer_lo == 0
    for op in (a, b):
        for l in range(3):
            op.set_level(l, init[l])
    a.apply_async(nt, 0)
    b.apply_async(nt, 0)
    sma, smb = a.collect(nt), b.collect(nt)
    assert a.stats().kernel_launches == nt and b.stats().kernel_launches == nt  # no ordering kernels
    got = np.zeros_like(ref)
    for l in range(3):
        la, lb = a.get_level(l), b.get_level(l)
        got[l, :50] = la[:50]
        got[l, 50:] = lb[50:]
    assert np.array_equal(got, ref)
    assert np.array_equal(np.maximum(sma, smb), r1.step_max_abs)
    a.close()
    b.close()


@needs2
def test_bench_two_gpus():
    p = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "50", "--warmup", "5",
                        "--no-sweep", "--no-cpu", "--e2e-reps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    line = [l for l in p.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == 2 and d["value"] > 0
    links = [l for l in p.stderr.splitlines() if l.startswith("[rank ")]
    assert len(links) == 2, p.stderr[-3000:]
    assert "upper: device 1 fused 1" in links[0] or "upper: device 1 fused 1" in links[1]
