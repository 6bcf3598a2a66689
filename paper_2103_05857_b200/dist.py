"""Multi-process plumbing for the column-sharded path.

One process per GPU (torch.distributed for rendezvous only). Every rank holds
one column shard of a sharded Solver; the per-step exchanges (the subtree
partials of the fixed 256-chunk sums, R19) run inside libsro.so as in-place
NCCL all-gathers on the solver stream (or, transport="host", through a host
all-gather callback over a torch.distributed group). This module only computes
which columns a rank holds, slices its inputs and shares the NCCL unique id or
wires the host all-gather.
"""
from __future__ import annotations

import numpy as np

from .sro import Solver, nccl_unique_id


def held_columns(n: int, shards: int, shard: int, shard_block: int = 0) -> np.ndarray:
    """Global indices (ascending) of the columns shard `shard` of `shards` holds:
    in every group of B_o = shard_block (0 -> n) consecutive columns, the
    shard-th contiguous B_o/shards of them (sro.h, sro_params.shard_block)."""
    Bo = n if shard_block == 0 else shard_block
    if shards < 1 or shards & (shards - 1) or n % Bo or Bo % shards:
        raise ValueError("shards must be a power of two dividing shard_block, which must divide n")
    Bl = Bo // shards
    p = np.arange(n // shards)
    return (p // Bl) * Bo + shard * Bl + p % Bl


def shard_cost_inputs(shards: int, shard: int, shard_block: int = 0, *, C=None, Y=None):
    """This shard's columns of a dense m x n cost and/or of the n x 3 target colours."""
    if C is None and Y is None:
        return None, None
    n = C.shape[1] if C is not None else Y.shape[0]
    cols = held_columns(n, shards, shard, shard_block)
    return (None if C is None else np.ascontiguousarray(C[:, cols]),
            None if Y is None else np.ascontiguousarray(Y[cols]))


def share_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank of `group` receives it."""
    import torch.distributed as dist
    box = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]


def host_allgather(group=None):
    """An exchange for sro_params.exchange over a torch.distributed group (e.g. gloo): the
    (nranks, count) host buffer's row `rank` is all-gathered into every row, in place."""
    import torch
    import torch.distributed as dist

    def f(buf, rank):
        rows = list(torch.from_numpy(buf).unbind(0))            # views into buf
        dist.all_gather(rows, torch.from_numpy(buf[rank].copy()), group=group)
    return f


def sharded_solver(a, b, lam, *, shard_block: int = 0, C=None, X=None, Y=None, cost="dense", group=None,
                   transport: str = "nccl", **kw) -> Solver:
    """A Solver holding this rank's column shard (collective over `group`).
    C / Y are the FULL cost / target colours; each rank passes on its columns only.
    transport: "nccl" (device all-gathers on the solver stream) or "host" (sro_params.exchange
    through `group`, e.g. gloo). Sequential BCFW-family variants do not shard (replicas only)."""
    import torch.distributed as dist
    G, rank = dist.get_world_size(group), dist.get_rank(group)
    Cl, Yl = shard_cost_inputs(G, rank, shard_block, C=C, Y=Y)
    if transport == "host":
        return Solver(a, b, lam, C=Cl, X=X, Y=Yl, cost=cost, shards=G, shard_block=shard_block, nranks=G,
                      rank=rank, exchange=host_allgather(group), **kw)
    uid = share_unique_id(group)
    return Solver(a, b, lam, C=Cl, X=X, Y=Yl, cost=cost, shards=G, shard_block=shard_block, nranks=G, rank=rank,
                  nccl_id=uid, **kw)
