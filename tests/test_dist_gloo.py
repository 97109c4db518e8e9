"""N>1 path on CPU: world_size-2 gloo process group exercising the sharding, the
max-over-ranks timing / summed-token reduction and the ordered output gather that
bench.py uses under torchrun (split by lines, merge in order)."""
import os

import numpy as np
import torch.multiprocessing as mp

from paper_2109_08008_b200.dist import (shard_range, chunk_index, reduce_timing, gather_outputs,
                                        gather_device_outputs, outputs_digest)


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


def _worker_dev(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 11
        lo, hi = shard_range(n, rank, world)
        stride = 6
        d_out = torch.full((hi - lo, stride), -7, dtype=torch.int32)
        d_len = torch.zeros(hi - lo, dtype=torch.int32)
        for k, i in enumerate(range(lo, hi)):
            L = i % 5
            d_out[k, :L] = torch.arange(L, dtype=torch.int32) + 100 * i
            d_len[k] = L
        res = gather_device_outputs(d_out, d_len)
        q.put((rank, None if res is None else (res[0].tolist(), res[1].tolist())))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_whole_set_gather():
    """C5 whole-set merge: contiguous shards over 3 ranks (uneven sizes), padded tensor
    all_gather, rank-order concatenation == the single-process outputs; digest equal."""
    world = 3
    port = 30500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_dev, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat, lens = res[0]
    exp_l = [i % 5 for i in range(11)]
    exp_t = [100 * i + k for i in range(11) for k in range(i % 5)]
    assert lens == exp_l and flat == exp_t
    assert res[1] is None and res[2] is None
    assert outputs_digest(np.array(flat), np.array(lens)) == \
        outputs_digest(np.array(exp_t, np.int32), np.array(exp_l, np.int32))
