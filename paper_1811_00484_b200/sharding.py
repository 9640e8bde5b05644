"""Multi-GPU component sharding (north star: Green's-tensor components sharded
across GPUs, NCCL over NVLink reducing the output currents).

Each rank holds the Tucker forms of its share of the canonical components, runs
the full pipeline (forward FFTs of every source current, fused Hadamard over
its components, inverse FFTs) and the partial output currents are summed with
one all-reduce of S * N_v complex values.  For apply_system only rank 0 adds
the eps * g * x diagonal term, so the reduced result is the exact system
matvec (the epilogue is linear in the component sum).
"""
from __future__ import annotations


def shard_components(ncomp: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment: balances the per-component block counts of the
    PWC/PWL tables (diagonal components, with fewer blocks, interleave with
    off-diagonal ones)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_components: bad rank/world")
    return [c for c in range(ncomp) if c % world == rank]


def allreduce_sum_(y, group=None):
    """In-place sum of the partial currents over the process group."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y


def sharded_apply_operator(op, x, out=None, group=None, stream=None):
    """apply_operator on a component-sharded operator + NCCL sum of the outputs."""
    from .vie import apply_operator

    y = apply_operator(op, x, out=out, stream=stream)
    return allreduce_sum_(y, group)


def sharded_apply_system(eps_r, inv_v, op, x, out=None, group=None, stream=None):
    import torch.distributed as dist

    from .vie import apply_system

    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    y = apply_system(eps_r, inv_v, op, x, out=out, diag_term=(rank == 0), stream=stream)
    return allreduce_sum_(y, group)
