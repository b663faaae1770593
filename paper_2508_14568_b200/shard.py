"""Multi-GPU plumbing for batches of independent pairs (cfg5-style).

Pairs are independent, so ranks split them with no data-path
collective: rank r takes pairs[r::world]; each GPU holds its own replica of
the keys. The only communication is the final gather of per-pair results
(a few bytes each) for reporting, over the torch.distributed process group
(NCCL on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def shard(items, rank: int, world: int):
    """The pairs this rank processes, with their global indices."""
    return [(i, items[i]) for i in range(rank, len(items), world)]


def gather_results(local, world: int, total: int):
    """local: list of (global_index, result). Returns the full list in order
    on every rank (all_gather_object: metadata only, never ciphertexts)."""
    import torch.distributed as dist
    if world == 1:
        out = [None] * total
        for i, r in local:
            out[i] = r
        return out
    parts = [None] * world
    dist.all_gather_object(parts, local)
    out = [None] * total
    for part in parts:
        for i, r in part:
            out[i] = r
    return out


def run_sharded(items, fn, rank: int, world: int):
    """fn(list_of_items) -> list_of_results, applied to this rank's shard."""
    mine = shard(items, rank, world)
    res = fn([it for _, it in mine]) if mine else []
    return gather_results(list(zip([i for i, _ in mine], res)), world, len(items))


def compute_batch_sharded(pairs, rank: int, world: int, ctx=None, _traverse=None, **kw):
    """cfg5-style batch across ranks: this rank runs compute_batch (one
    wavefront on its own GPU and key replica) over pairs[rank::world];
    every rank returns all reports in input order (gathered as plain dicts,
    never ciphertexts). The reference's own concurrency is one thread per
    pair (cli.cpp:194-207); here each rank's shard is one launch sequence."""
    from . import leuven
    return run_sharded(pairs, lambda ps: leuven.compute_batch(ps, ctx=ctx, _traverse=_traverse, **kw),
                       rank, world)
