"""Multi-process z-slab decomposition through CUDA IPC (one process per slab; on a 1-GPU
box the processes share the device, which exercises the same IPC + peer-store + flag path
as one-GPU-per-process over NVLink).  N slabs must equal 1 domain bit for bit."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("form", ["factorised", "plain_f64"])
def test_multiprocess_slabs_bitwise(world, form):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + world * 7 + (form == 'factorised')}",
           os.path.join(ROOT, "scripts", "mp_slab_check.py"), form]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "MP_SLAB_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]


def test_multiprocess_slabs_bitwise_so16_pencil():
    """The SO 16 K1 variant with the y-pencil warp (forced) across two IPC-linked processes."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29571",
           os.path.join(ROOT, "scripts", "mp_slab_check.py"), "factorised", "16"]
    env = dict(os.environ, SWB_YW="1", SWB_T1="20")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    assert "MP_SLAB_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-2000:]
