"""Multi-process (gloo, world_size 2 and 4) check of the ns2d / ns3d slab
decomposition's host-side logic: partitions, block layouts and the two
all-to-all transposes (tests/dist_slab_np.py mirrors csrc/skgpu.cu and the
fast-path kernels' indexing) against the undecomposed oracle tendency."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import spectral_np as O
from paper_1807_01769_b200 import ic


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out):
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    sys.path[:0] = [str(here), str(here.parent)]
    import torch.distributed as dist
    from dist_slab_np import slab_tendency
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = ic.ns2d_ic(n, seed=5)
    N, c0, c1 = slab_tendency(w, n, rank, world)
    ref = O.tendency_ns2d(w, n)[0][:, c0:c1]
    out[rank] = O.rel_l2(N, ref) if np.linalg.norm(ref) > 0 else float(np.abs(N).max())
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, (64, 64)), (4, (128, 64)), (2, (32, 128)), (4, (64, 64))])
def test_slab_decomposition_gloo(world, n):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _port(), n, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        assert out[r] < 1e-12, (r, out[r])


def _worker3(rank, world, port, n, out):
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    sys.path[:0] = [str(here), str(here.parent)]
    import torch.distributed as dist
    from dist_slab_np import slab3d_tendency
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v = ic.ns3d_ic(n, seed=5)
    N, gky, kzc = slab3d_tendency(v, n, rank, world)
    ref = O.tendency_ns3d(v, n)[:, :, gky, :kzc]
    out[rank] = max(O.rel_l2(N[c], ref[c]) for c in range(3))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, (16, 16, 16)), (4, (16, 32, 16)), (2, (32, 16, 8))])
def test_slab3d_decomposition_gloo(world, n):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker3, args=(world, _port(), n, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        assert out[r] < 1e-12, (r, out[r])


def _worker_pencil(rank, world, port, n, grid, out):
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    sys.path[:0] = [str(here), str(here.parent)]
    import torch.distributed as dist
    from dist_slab_np import pencil3d_tendency, pencil_groups
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    py, pz = grid
    groups = pencil_groups(py, pz)
    v = ic.ns3d_ic(n, seed=5)
    N, gky, (k0, k1) = pencil3d_tendency(v, n, rank, py, pz, groups)
    ref = O.tendency_ns3d(v, n)[:, :, gky, k0:k1]
    nrm = max(np.linalg.norm(ref[c]) for c in range(3))
    out[rank] = max(np.linalg.norm(N[c] - ref[c]) for c in range(3)) / nrm
    dist.destroy_process_group()


@pytest.mark.parametrize("grid,n", [((2, 2), (16, 16, 16)), ((1, 2), (16, 16, 32)), ((2, 1), (16, 16, 16)),
                                    ((2, 2), (16, 32, 16))])
def test_pencil3d_decomposition_gloo(grid, n):
    """ns3d pencil decomposition (py x pz process grid, two all-to-alls per
    3D FFT inside the ky / x and the kz / y sub-communicators) against the
    undecomposed oracle tendency, one process per part."""
    world = grid[0] * grid[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_pencil, args=(world, _port(), n, grid, out), nprocs=world, join=True)
    assert len(out) == world
    for r in range(world):
        assert out[r] < 1e-12, (r, out[r])
