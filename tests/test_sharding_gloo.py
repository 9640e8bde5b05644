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


# --------------------------------------------------------------------------
# Slab decomposition host logic (vie_slab_* dataflow) with real gloo all-to-alls:
# the per-rank stages are numpy stand-ins for the three C-ABI stages using the same
# rank-blocked exchange layout [rank][s][k in block][axis-2 row in block][axis-1].
def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_1811_00484_b200.sharding import local_slab, slab_planes
    from tests.helpers import fourier_forms, random_field, spatial_tucker_forms

    kind, basis, dims = 0, 0, (12, 4, 6)
    n1, n2, n3 = dims
    m1, m2, m3 = 2 * n1, 2 * n2, 2 * n3
    S = 3
    spatial, par = spatial_tucker_forms(kind, basis, dims, 2, 4)
    forms = fourier_forms(spatial, par)
    _, _, blocks = orc.component_table(kind, basis)
    spec = [orc.decompress_tucker((m1, m2, m3), f).reshape(m3, m2, m1) for f in forms]
    x = random_field(basis, dims, 8)
    k0, nk = slab_planes(n3, rank, world)
    W = m1 // world
    xl = local_slab(x, S, n3, n1 * n2, rank, world).reshape(S, nk, n2, n1)
    # stage 1: axis-1 FFT of the local z-slab, blocked by the destination rank's W positions
    xa = np.zeros((S, nk, n2, m1), complex)
    xa[..., :n1] = xl
    xa = np.fft.fft(xa, axis=3)
    send = np.stack([xa[..., qq * W:(qq + 1) * W] for qq in range(world)]).reshape(-1)
    recv = torch.empty(send.size, dtype=torch.complex128)
    dist.all_to_all_single(recv, torch.from_numpy(send))
    # stage 2: this rank's W positions, all k: axis-2 FFT, axis-3 FFT, Hadamard, inverses
    blk = recv.numpy().reshape(world, S, nk, n2, W)
    xp = np.zeros((S, m3, m2, W), complex)
    xp[:, :n3, :n2] = blk.transpose(1, 0, 2, 3, 4).reshape(S, n3, n2, W)
    xp = np.fft.fft(np.fft.fft(xp, axis=2), axis=1)
    cols = slice(rank * W, (rank + 1) * W)
    yp = np.zeros_like(xp)
    for t, s_, c, coef in blocks:
        yp[t] += coef * spec[c][:, :, cols] * xp[s_]
    yp = np.fft.ifft(np.fft.ifft(yp, axis=1)[:, :n3], axis=2)[:, :, :n2]
    out = np.stack([yp[:, r * nk:(r + 1) * nk] for r in range(world)]).reshape(-1)
    back = torch.empty(out.size, dtype=torch.complex128)
    dist.all_to_all_single(back, torch.from_numpy(out))
    # stage 3: inverse axis-1 FFT of the local z-slab rows, crop
    ya = back.numpy().reshape(world, S, nk, n2, W).transpose(1, 2, 3, 0, 4).reshape(S, nk, n2, m1)
    yl = np.fft.ifft(ya, axis=3)[..., :n1]
    gathered = [torch.empty(yl.size, dtype=torch.complex128) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(np.ascontiguousarray(yl).reshape(-1)))
    if rank == 0:
        y = np.concatenate([g.numpy().reshape(S, nk, n1 * n2) for g in gathered], axis=1).reshape(-1)
        ref = orc.apply_operator_tucker(kind, basis, dims, forms, x)
        q.put(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
