"""CPU, world size 2 over gloo: the pair-sharding path used for multi-GPU
batches (shard.compute_batch_sharded -> leuven.compute_batch on each rank's
shard, then the gather) splits the cfg5 pairs without overlap and returns
every report in order. Only the innermost GPU traversal (encrypt + one
wavefront + decrypt, leuven._traverse_batch) is stubbed — by the plaintext
Wagner-Fischer distance and the C library's own symbolic plan (lv_plan_trace,
no device work) for the counters — so report assembly, sharding and gather
are the product code."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2508_14568_b200 import shard, workloads as W
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2508_14568_b200 import leuven as LV
    pairs = W.cfg5(32)
    seen = [i for i, _ in shard.shard(pairs, rank, world)]

    def traverse(ctx, ps, spec, bands, key_encoding):  # the GPU part, stubbed
        out = []
        for (a, b), band in zip(ps, bands):
            _, tot = LV.plan_trace(len(a), len(b), band, key_encoding, 4000.0)
            tot.equality_pbs = tot.visited_cells * spec.symbol_count()
            out.append((W.wf_distance(a, b) % 32, tot))
        return out
    res = shard.compute_batch_sharded(pairs, rank, world, _traverse=traverse)
    q.put((rank, seen, res))
    dist.barrier()
    dist.destroy_process_group()


def test_pair_sharding_gloo_world2(golden):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    seen = sorted(i for _, s, _ in out for i in s)
    assert seen == list(range(32))  # disjoint and complete
    want = [c["report"] for c in golden["configs"]["cfg5"][:32]]
    for _, _, res in out:
        assert len(res) == 32
        for got, w in zip(res, want):
            for f in ("distance", "half_width", "visited_cells", "pbs_total", "pbs_equality",
                      "pbs_kernel", "refresh_count", "preprocessing_pbs", "max_key_variance"):
                assert got[f] == w[f], (f, got[f], w[f])
