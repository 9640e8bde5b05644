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
# Slab decomposition host logic with real gloo all-to-alls: the product's SlabMatvec class
# (sharding.py: buffers, stage order, the two exchanges over torch.distributed) runs with its
# three library stages replaced by numpy stand-ins that use the same rank-blocked exchange
# layout [rank][s][k in block][axis-2 row in block][axis-1] as vie_slab_forward / _pencil /
# _inverse (the GPU emulation test, test_gpu_slab.py, checks the real stages on that layout).
def _numpy_slab_class():
    from paper_1811_00484_b200.sharding import SlabMatvec

    class NumpySlab(SlabMatvec):
        def __init__(self, rank, world, dims, S, spec, blocks):
            self.dims, self.S, self.spec, self.blocks = dims, S, spec, blocks
            n1, n2, n3 = dims
            self.nkv, self.W = n3 // world, 2 * n1 // world
            import types

            super().__init__(types.SimpleNamespace(), rank, world)

        def _partition(self):
            n1, n2, n3 = self.dims
            return (self.S * n1 * n2 * self.nkv, self.S * self.nkv * n2 * 2 * n1, self.rank * self.nkv, self.nkv)

        def _empty(self, n):
            return torch.empty(n, dtype=torch.complex128)

        def forward(self, x_local, stream=None):  # stand-in for vie_slab_forward
            n1, n2, n3 = self.dims
            m1 = 2 * n1
            xa = np.zeros((self.S, self.nk, n2, m1), complex)
            xa[..., :n1] = x_local.numpy().reshape(self.S, self.nk, n2, n1)
            xa = np.fft.fft(xa, axis=3)
            W = self.W
            send = np.stack([xa[..., q * W:(q + 1) * W] for q in range(self.world)]).reshape(-1)
            self.send.copy_(torch.from_numpy(send))

        def pencil(self, stream=None):  # stand-in for vie_slab_pencil
            n1, n2, n3 = self.dims
            m1, m2, m3 = 2 * n1, 2 * n2, 2 * n3
            S, W, nk, world = self.S, self.W, self.nk, self.world
            blk = self.recv.numpy().reshape(world, S, nk, n2, W)
            xp = np.zeros((S, m3, m2, W), complex)
            xp[:, :n3, :n2] = blk.transpose(1, 0, 2, 3, 4).reshape(S, n3, n2, W)
            xp = np.fft.fft(np.fft.fft(xp, axis=2), axis=1)
            cols = slice(self.rank * W, (self.rank + 1) * W)
            yp = np.zeros_like(xp)
            for t, s_, c, coef in self.blocks:
                yp[t] += coef * self.spec[c][:, :, cols] * xp[s_]
            yp = np.fft.ifft(np.fft.ifft(yp, axis=1)[:, :n3], axis=2)[:, :, :n2]
            out = np.stack([yp[:, r * nk:(r + 1) * nk] for r in range(world)]).reshape(-1)
            self.out.copy_(torch.from_numpy(out))

        def inverse(self, y_local, eps_local=None, inv_v=0.0, x_local=None, diag=True, stream=None):
            n1, n2, n3 = self.dims
            ya = self.back.numpy().reshape(self.world, self.S, self.nk, n2, self.W)
            ya = ya.transpose(1, 2, 3, 0, 4).reshape(self.S, self.nk, n2, 2 * n1)
            y_local.copy_(torch.from_numpy(np.ascontiguousarray(np.fft.ifft(ya, axis=3)[..., :n1]).reshape(-1)))

    return NumpySlab


def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as orc
    from paper_1811_00484_b200.sharding import local_slab
    from tests.helpers import fourier_forms, random_field, spatial_tucker_forms

    kind, basis, dims = 0, 0, (12, 4, 6)
    n1, n2, n3 = dims
    S = 3
    spatial, par = spatial_tucker_forms(kind, basis, dims, 2, 4)
    forms = fourier_forms(spatial, par)
    _, _, blocks = orc.component_table(kind, basis)
    spec = [orc.decompress_tucker((2 * n1, 2 * n2, 2 * n3), f).reshape(2 * n3, 2 * n2, 2 * n1) for f in forms]
    x = random_field(basis, dims, 8)
    sm = _numpy_slab_class()(rank, world, dims, S, spec, blocks)
    assert sm.op.local_elems == sm.x_elems and sm.k0 == rank * (n3 // world)
    xl = torch.from_numpy(np.ascontiguousarray(local_slab(x, S, n3, n1 * n2, rank, world)))
    yl = sm.apply(xl)  # the product's apply(): forward -> all_to_all -> pencil -> all_to_all -> inverse
    gathered = [torch.empty(yl.numel(), dtype=torch.complex128) for _ in range(world)]
    dist.all_gather(gathered, yl)
    if rank == 0:
        y = np.concatenate([g.numpy().reshape(S, n3 // world, n1 * n2) for g in gathered], axis=1).reshape(-1)
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
