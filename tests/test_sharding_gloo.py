"""World-size-2 gloo test of the multi-GPU host logic on CPU: component shards
computed per rank (oracle as the per-rank compute stand-in: forms of the other
ranks' components are zero) and summed with an all-reduce equal the full
matvec / system matvec."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_00484_b200.sharding import shard_components


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, basis, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from tests.helpers import fourier_forms, random_field, spatial_tucker_forms

    dims = (3, 4, 3)
    spatial, par = spatial_tucker_forms(0, basis, dims, 2, 9)
    nc = len(spatial)
    mine = set(shard_components(nc, rank, world))
    masked = [(core if c in mine else np.zeros_like(core), us) for c, (core, us) in enumerate(spatial)]
    forms = fourier_forms(masked, par)
    x = random_field(basis, dims, 1)
    y = torch.from_numpy(orc.apply_operator_tucker(0, basis, dims, forms, x))
    dist.all_reduce(y)
    nv = int(np.prod(dims))
    eps = 2.0 + 0.5j + np.arange(nv) / nv
    # system matvec: only rank 0 carries the diagonal term
    ys = orc.apply_system_tucker(basis, dims, forms, eps, 0.3, x)
    if rank != 0:
        S = orc.ncur(basis)
        g = np.array([1.0 if (basis == 0 or s % 4 == 0) else 1 / 12 for s in range(S)])
        ys = ys - np.concatenate([eps * g[s] * x[s * nv:(s + 1) * nv] for s in range(S)])
    ys = torch.from_numpy(ys)
    dist.all_reduce(ys)
    if rank == 0:
        full = fourier_forms(spatial, par)
        ref = orc.apply_operator_tucker(0, basis, dims, full, x)
        refs = orc.apply_system_tucker(basis, dims, full, eps, 0.3, x)
        q.put((np.linalg.norm(y.numpy() - ref) / np.linalg.norm(ref),
               np.linalg.norm(ys.numpy() - refs) / np.linalg.norm(refs)))
    dist.destroy_process_group()


@pytest.mark.parametrize("basis", [0, 1])
def test_component_shards_allreduce_to_full(basis):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, basis, q)) for r in range(2)]
    for p in procs:
        p.start()
    e1, e2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert e1 < 1e-13 and e2 < 1e-13


def test_shard_assignment_partitions():
    for nc in (3, 6, 30, 60):
        for world in (1, 2, 4, 8):
            got = sorted(c for r in range(world) for c in shard_components(nc, r, world))
            assert got == list(range(nc))
    with pytest.raises(ValueError):
        shard_components(6, 2, 2)
