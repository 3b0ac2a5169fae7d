"""Multi-GPU plumbing for the independent-unit workloads:
batched energy rows and FMO fragments are sharded across ranks with no
data-path collective; only the scalar energies are gathered, in fixed order.

One process per GPU (torchrun); torch.distributed is the transport (NCCL on
the GPU box, gloo in the CPU tests). The sharding decisions are the C++ host
API's (shard_by_cost), so every rank computes the same assignment.
"""
from __future__ import annotations

import numpy as np

from . import assemble_fragments, fragment_cost, shard_by_cost


def row_range(n_rows: int, rank: int, world: int):
    """Contiguous block of rows for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_rows, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local: np.ndarray, n_rows: int, group=None):
    """All-gather per-rank row blocks back into rank order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, np.asarray(local, np.float64), group=group)
    out = np.concatenate(parts)
    assert out.shape[0] == n_rows
    return out


def fragment_owners(fragments, world: int):
    return shard_by_cost([fragment_cost(f) for f in fragments], world)


def fmo_energy(fragments, n_fragments: int, evaluate, group=None):
    """FMO two-body energy with fragments sharded over the process group.

    `evaluate(fragments, rank, world) -> {label: energy}` computes this rank's
    share (the C++ evaluate_fragments on a device, or a CPU checker in tests).
    Returns (assembled energy, {label: energy}) identically on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = evaluate(fragments, rank, world)
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, mine, group=group)
    else:
        parts = [mine]
    energies = {}
    for p in parts:  # fixed rank order; labels are disjoint across ranks
        energies.update(p)
    return assemble_fragments(n_fragments, energies), energies
