"""N>1 path on CPU: world_size-2 gloo process group exercising the sharding, the
max-over-ranks timing / summed-token reduction and the ordered output gather that
bench.py uses under torchrun (split by lines, merge in order)."""
import os

import numpy as np
import torch.multiprocessing as mp

from paper_2109_08008_b200.dist import shard_range, chunk_index, reduce_timing, gather_outputs


def test_shard_range_covers_exactly_once():
    for n in (0, 1, 7, 1000, 2998):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            sizes = [hi - lo for lo, hi in got]
            assert max(sizes) - min(sizes) <= 1


def test_chunk_index_disjoint():
    seen = {chunk_index(k, r, 4) for k in range(5) for r in range(4)}
    assert len(seen) == 20


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ms, tok = reduce_timing(10.0 + rank, 100.0 * (rank + 1))
        # every rank translated its contiguous shard of 7 fake "sentences"
        lo, hi = shard_range(7, rank, world)
        outs = [[i] * (i % 3) for i in range(lo, hi)]
        merged = gather_outputs(outs)
        q.put((rank, ms, tok, merged))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reduce_and_gather():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ms, tok, merged in res:
        assert ms == 11.0            # max over ranks
        assert tok == 300.0          # sum over ranks
        if rank == 0:
            assert merged == [[i] * (i % 3) for i in range(7)]   # original order restored
        else:
            assert merged is None
