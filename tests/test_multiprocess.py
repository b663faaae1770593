"""CPU, world size 2 over gloo: the pair-sharding path used for multi-GPU
batches splits the cfg5 pairs without overlap and gathers every result in
order. The per-pair compute here is the plaintext Wagner-Fischer stand-in
(no GPU on this box); on the GPU box the same code runs compute_batch."""
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
    pairs = W.cfg5(32)
    seen = [i for i, _ in shard.shard(pairs, rank, world)]
    res = shard.run_sharded(pairs, lambda ps: [W.wf_distance(a, b) for a, b in ps], rank, world)
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
    want = [c["report"]["distance"] for c in golden["configs"]["cfg5"][:32]]
    for _, _, res in out:
        assert res == want
