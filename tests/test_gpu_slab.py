"""Slab-decomposed multi-GPU matvec: z-slabs for the axis-1 passes, axis-1
position slabs for the axis-2 passes / decomposition / pencil stage, one all-to-all each
way after the axis-1 FFT; emulated rank by rank on one GPU:
every rank's stage runs to completion before the exchange (no rank waits on
another inside a kernel), the all-to-all is done by chunk copies with the exact
semantics of torch.distributed.all_to_all_single.  The assembled result must equal
the single-GPU matvec."""
import numpy as np
import pytest

from tests.helpers import random_field, rel
from tests.test_gpu_parity import K, N, PWC, PWL, make_ops, vie, dft  # noqa: F401

pytestmark = pytest.mark.gpu


def _emulate(vie, ops, xg, dims, S, world, eps=None, inv_v=0.0):
    import torch

    from paper_1811_00484_b200.sharding import SlabMatvec, local_slab

    n1, n2, n3 = dims
    sms = [SlabMatvec(ops[r], r, world) for r in range(world)]
    xs = [local_slab(xg, S, n3, n1 * n2, r, world).contiguous() for r in range(world)]
    es = None
    if eps is not None:
        es = [local_slab(eps, 1, n3, n1 * n2, r, world).contiguous() for r in range(world)]
    for r in range(world):
        sms[r].forward(xs[r])
    torch.cuda.synchronize()
    for q in range(world):  # recv_q[chunk r] = send_r[chunk q]
        for r in range(world):
            sms[q].recv.view(world, -1)[r].copy_(sms[r].send.view(world, -1)[q])
    for q in range(world):
        sms[q].pencil()
    torch.cuda.synchronize()
    for r in range(world):
        for q in range(world):
            sms[r].back.view(world, -1)[q].copy_(sms[q].out.view(world, -1)[r])
    ys = []
    for r in range(world):
        y = torch.empty_like(xs[r])
        sms[r].inverse(y, None if es is None else es[r], inv_v, xs[r] if es is not None else None, True)
        ys.append(y)
    torch.cuda.synchronize()
    nk = n3 // world
    return torch.cat([y.view(S, nk, n1 * n2) for y in ys], dim=1).reshape(-1)


SLAB_CASES = [
    (N, PWL, (4, 4, 8), 2, 3), (N, PWL, (4, 4, 8), 4, 3), (N, PWC, (16, 8, 8), 4, 4), (K, PWL, (6, 4, 6), 2, 3),
    (N, PWL, (4, 4, 32), 4, 3), (N, PWC, (32, 3, 64), 8, 3), (K, PWC, (8, 6, 10), 2, 3), (N, PWC, (4, 4, 4), 1, 2),
]


@pytest.mark.parametrize("kind,basis,dims,world,rank", SLAB_CASES)
def test_slab_ranks_assemble_the_single_gpu_matvec(vie, dft, orc, kind, basis, dims, world, rank):
    import torch

    S = 3 if basis == PWC else 12
    x = torch.from_numpy(random_field(basis, dims, 300 + world)).cuda()
    op1, oforms, _, _ = make_ops(vie, dft, orc, kind, basis, dims, rank, 21 + sum(dims))
    y_ref = vie.apply_operator(op1, x)
    ops = [make_ops(vie, dft, orc, kind, basis, dims, rank, 21 + sum(dims))[0] for _ in range(world)]
    y = _emulate(vie, ops, x, dims, S, world)
    assert rel(y_ref.cpu().numpy(), y.cpu().numpy()) <= 1e-13, (kind, basis, dims, world)
    assert rel(orc.apply_operator_tucker(kind, basis, dims, oforms, x.cpu().numpy()), y.cpu().numpy()) <= 1e-10


def test_slab_system_matvec(vie, dft, orc):
    import torch

    dims, world = (6, 4, 6), 3
    x = torch.from_numpy(random_field(PWL, dims, 9)).cuda()
    rng = np.random.default_rng(3)
    eps = torch.from_numpy(1 + rng.random(int(np.prod(dims))) + 0.3j * rng.random(int(np.prod(dims)))).cuda()
    op1 = make_ops(vie, dft, orc, N, PWL, dims, 3, 77)[0]
    y_ref = vie.apply_system(eps, 0.7, op1, x)
    ops = [make_ops(vie, dft, orc, N, PWL, dims, 3, 77)[0] for _ in range(world)]
    y = _emulate(vie, ops, x, dims, 12, world, eps=eps, inv_v=0.7)
    assert rel(y_ref.cpu().numpy(), y.cpu().numpy()) <= 1e-13


def test_partition_errors_and_guard(vie, dft, orc):
    import torch

    from paper_1811_00484_b200.sharding import SlabMatvec

    dims = (8, 6, 8)
    op = make_ops(vie, dft, orc, N, PWC, dims, 2, 5)[0]
    with pytest.raises(ValueError):
        SlabMatvec(op, 0, 3)  # n3 = 8 not divisible by 3
    with pytest.raises(ValueError):
        SlabMatvec(op, 0, 4)  # 2 n1 = 16 positions give 4 per rank: not a whole PWC pencil group (8)
    SlabMatvec(op, 1, 2)
    with pytest.raises(ValueError):  # a partitioned operator refuses the unpartitioned matvec
        vie.apply_operator(op, torch.zeros(3 * int(np.prod(dims)), dtype=torch.complex128, device="cuda"))


def test_library_exchange_and_distributed_gmres_single_rank(vie, dft, orc):
    """The in-library multi-GPU path (vie_comm over NCCL, vie_slab_matvec, vie_gmres_solve on a
    partitioned operator with all-reduced dots) on a one-rank communicator: the grouped
    send/recv exchange, the side-stream decomposition and the NCCL all-reduce hook all run;
    results equal the single-GPU path."""
    import torch

    from paper_1811_00484_b200.sharding import SlabMatvec, make_comm

    dims = (6, 4, 6)
    nv = int(np.prod(dims))
    x = torch.from_numpy(random_field(PWL, dims, 41)).cuda()
    rng = np.random.default_rng(8)
    eps = torch.from_numpy(2 + rng.random(nv) + 0.3j * rng.random(nv)).cuda()
    op1 = make_ops(vie, dft, orc, N, PWL, dims, 3, 19, scale=0.05)[0]
    op = make_ops(vie, dft, orc, N, PWL, dims, 3, 19, scale=0.05)[0]
    comm = make_comm(dft, 0, 1)
    sm = SlabMatvec(op, 0, 1, comm=comm)
    assert sm.send is None  # no Python-side exchange buffers: the library owns them
    y = sm.apply(x)
    assert rel(vie.apply_operator(op1, x).cpu().numpy(), y.cpu().numpy()) <= 1e-13
    ys = sm.apply(x, eps_local=eps, inv_v=0.7)
    assert rel(vie.apply_system(eps, 0.7, op1, x).cpu().numpy(), ys.cpu().numpy()) <= 1e-13
    rhs = torch.from_numpy(random_field(PWL, dims, 42)).cuda()
    cfg = vie.GmresConfig(1e-10, 20, 3)
    r1 = vie.gmres(op1, eps, 0.7, rhs, cfg)
    r2 = vie.gmres(op, eps, 0.7, rhs, cfg)
    assert r1.iterations == r2.iterations and r1.converged == r2.converged
    assert np.max(np.abs(np.array(r1.residual_history) - np.array(r2.residual_history))
                  / np.array(r1.residual_history)) <= 1e-10
    assert rel(r1.solution.cpu().numpy(), r2.solution.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("world,dims,basis", [(2, (6, 4, 6), PWL), (3, (6, 4, 6), PWL), (4, (4, 4, 8), PWL),
                                              (2, (8, 6, 10), PWC)])
def test_library_slab_matvec_and_distributed_gmres_loopback(vie, dft, orc, world, dims, basis):
    """vie_slab_matvec and the distributed vie_gmres_solve at R > 1: R ranks as R host threads of
    this process on one GPU, each with its own context, operator and loopback communicator (the
    library's exchange and all-reduce paths with device copies between host barriers instead of
    NCCL -- no kernel waits on another rank).  The assembled result equals the single-GPU path."""
    import threading

    import torch

    from paper_1811_00484_b200.sharding import SlabMatvec, local_slab

    S = 3 if basis == PWC else 12
    n1, n2, n3 = dims
    nv = int(np.prod(dims))
    x = torch.from_numpy(random_field(basis, dims, 61)).cuda()
    rng = np.random.default_rng(12)
    eps = torch.from_numpy(2 + rng.random(nv) + 0.3j * rng.random(nv)).cuda()
    rhs = torch.from_numpy(random_field(basis, dims, 62)).cuda()
    op1 = make_ops(vie, dft, orc, N, basis, dims, 3, 23, scale=0.05)[0]
    y_ref = vie.apply_operator(op1, x)
    ys_ref = vie.apply_system(eps, 0.7, op1, x)
    cfg = vie.GmresConfig(1e-10, 12, 2)
    g_ref = vie.gmres(op1, eps, 0.7, rhs, cfg)
    lb = vie.Loopback(world)
    dfts = [vie.DftService(0) for _ in range(world)]
    ops = [make_ops(vie, dfts[r], orc, N, basis, dims, 3, 23, scale=0.05)[0] for r in range(world)]
    comms = [vie.Comm(dfts[r], world, r, loopback=lb) for r in range(world)]
    sms = [SlabMatvec(ops[r], r, world, comm=comms[r]) for r in range(world)]
    xs = [local_slab(x, S, n3, n1 * n2, r, world).contiguous() for r in range(world)]
    es = [local_slab(eps, 1, n3, n1 * n2, r, world).contiguous() for r in range(world)]
    bs = [local_slab(rhs, S, n3, n1 * n2, r, world).contiguous() for r in range(world)]
    out, errs = [None] * world, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            y = sms[r].apply(xs[r])
            ys = sms[r].apply(xs[r], eps_local=es[r], inv_v=0.7)
            g = vie.gmres(ops[r], es[r], 0.7, bs[r], cfg)
            torch.cuda.synchronize()
            out[r] = (y, ys, g)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    nk = n3 // world
    cat = lambda vs: torch.cat([v.view(S, nk, n1 * n2) for v in vs], dim=1).reshape(-1).cpu().numpy()
    assert rel(y_ref.cpu().numpy(), cat([o[0] for o in out])) <= 1e-13
    assert rel(ys_ref.cpu().numpy(), cat([o[1] for o in out])) <= 1e-13
    for o in out:  # every rank reports the same (global) iteration history
        assert o[2].iterations == g_ref.iterations and o[2].converged == g_ref.converged
        assert np.max(np.abs(np.array(o[2].residual_history) - np.array(g_ref.residual_history))
                      / np.array(g_ref.residual_history)) <= 1e-9
    assert rel(g_ref.solution.cpu().numpy(), cat([o[2].solution for o in out])) <= 1e-9
