"""Host-side logic of the z-slab decomposition on CPU with torch.distributed/gloo,
world_size 2 (the device-side halo exchange is covered by the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1912_00695_b200 import dist as D


def test_slab_bounds_partition():
    for n0 in (16, 64, 257, 2048):
        for world in (1, 2, 3, 4, 8):
            s = D.all_slabs(n0, world)
            assert s[0][0] == 0 and s[-1][1] == n0
            assert all(a[1] == b[0] for a, b in zip(s[:-1], s[1:]))
            sizes = [hi - lo for lo, hi in s]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.check_slabs(10, 4, 4)
    D.check_slabs(64, 8, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n0 = 12
        slab = D.slab_bounds(n0, world, rank)
        full = np.full((n0, 3, 4), 100.0 + rank, np.float32)
        lvl = D.gather_level(full, slab)
        smax = np.array([1.0 + rank, 5.0, np.nan if rank == 1 else 2.0], np.float32)
        red = D.reduce_step_max(smax)
        tr = np.zeros((2, 3), np.float32)
        tr[:, rank] = rank + 1.5
        trr = D.reduce_traces(tr)
        q.put((rank, lvl, red, trr))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lvl, red, trr in out:
        assert np.array_equal(lvl[:6], np.full((6, 3, 4), 100.0, np.float32))
        assert np.array_equal(lvl[6:], np.full((6, 3, 4), 101.0, np.float32))
        assert red[0] == 2.0 and red[1] == 5.0 and np.isnan(red[2])
        assert np.array_equal(trr, np.array([[1.5, 2.5, 0], [1.5, 2.5, 0]], np.float32))
