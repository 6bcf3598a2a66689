"""The N > 1 host path on CPU: world_size-2 gloo process groups (no GPU).

Covers what the sharded path does outside the kernels: the column ownership
map (sro.h shard_block), the slicing of each rank's inputs, the sharing of the
NCCL unique id, and — through a real 2-process exchange — the property every
sharded reduction relies on: per-rank subtrees of the fixed 256-chunk sum
(R19), all-gathered and combined by adjacent pairs, equal the single-process
sum bit for bit (computed by the oracle's chunk_tree_sum).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_05857_b200.dist import held_columns, shard_cost_inputs



def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _pair_tree(v):
    v = list(v)
    while len(v) > 1:
        v = [v[2 * c] + v[2 * c + 1] for c in range(len(v) // 2)]
    return v[0]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        from oracle import chunk_tree_sum
        from paper_2103_05857_b200.dist import share_unique_id
        res = {}
        # 1. the NCCL id created on rank 0 reaches every rank unchanged
        uid = share_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        res["id_ok"] = len(uid) == 128 and all(x == ids[0] for x in ids)
        # 2. subtree decomposition of the 256-chunk sum over U's positions
        ok = True
        for L, seed in [(256, 0), (1024, 1), (4096, 2), (65536, 3)]:
            x = np.random.default_rng(seed).standard_normal(L) * 10.0 ** np.random.default_rng(seed + 7).integers(
                -8, 8, L)
            lo, hi = rank * L // world, (rank + 1) * L // world
            mine = chunk_tree_sum(x[lo:hi], 256 // world)
            t = torch.tensor([mine], dtype=torch.float64)
            allv = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allv, t)
            combined = _pair_tree([float(v.item()) for v in allv])
            ok &= combined == chunk_tree_sum(x, 256)
        res["tree_ok"] = bool(ok)
        # 3. per-row subtrees of a block: rank r holds the block positions [r B/G, (r+1) B/G)
        B, m = 512, 64
        rng = np.random.default_rng(11)
        contrib = np.where(rng.random((B, m)) < 0.05, rng.standard_normal((B, m)), 0.0)
        lo, hi = rank * B // world, (rank + 1) * B // world
        sub = np.array([chunk_tree_sum(contrib[lo:hi, k], 256 // world) for k in range(m)])
        allv = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, torch.from_numpy(sub))
        comb = np.array([_pair_tree([float(v[k]) for v in allv]) for k in range(m)])
        ref = np.array([chunk_tree_sum(contrib[:, k], 256) for k in range(m)])
        res["rows_ok"] = bool(np.array_equal(comb, ref))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert out[r] == {"id_ok": True, "tree_ok": True, "rows_ok": True}, out


@pytest.mark.parametrize("n,G,Bo", [(256, 2, 0), (512, 4, 64), (8192, 8, 1024), (64, 1, 0)])
def test_held_columns_partition(n, G, Bo):
    """The G shards' held columns partition [n]; inside every ownership block each
    shard holds one contiguous run of B_o/G columns, in shard order."""
    parts = [held_columns(n, G, s, Bo) for s in range(G)]
    allc = np.sort(np.concatenate(parts))
    assert np.array_equal(allc, np.arange(n))
    B = n if Bo == 0 else Bo
    for s, p in enumerate(parts):
        assert np.all(np.diff(p) > 0)
        assert np.all((p % B) // (B // G) == s)


def test_held_columns_rejects_bad_layouts():
    with pytest.raises(ValueError):
        held_columns(256, 3, 0)
    with pytest.raises(ValueError):
        held_columns(256, 4, 0, 6)


def test_shard_cost_inputs_slices_columns():
    C = np.arange(6 * 16, dtype=np.float32).reshape(6, 16)
    Y = np.arange(16 * 3, dtype=np.float64).reshape(16, 3)
    Cl, Yl = shard_cost_inputs(4, 2, 8, C=C, Y=Y)
    cols = held_columns(16, 4, 2, 8)
    assert np.array_equal(cols, [4, 5, 12, 13])
    assert np.array_equal(Cl, C[:, cols]) and np.array_equal(Yl, Y[cols])
