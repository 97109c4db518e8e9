"""-m gpu: the C5 whole-set path with two ranks on the box's one GPU (gloo process group:
the ranks never wait on each other's kernels — each translates its own contiguous shard —
so sharing cuda:0 is safe; NCCL needs one GPU per rank).  The merged outputs (rank-order
all_gather) are byte-identical to one process translating the whole set."""
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N = 3000


def _rank(rank, world, port, q):
    import torch.distributed as dist
    from synth import newstest_like
    from gpu_common import gpu_model
    from paper_2109_08008_b200.dist import shard_range, gather_device_outputs, outputs_digest
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        full = newstest_like(N, 32000, start=40000)
        lo, hi = shard_range(N, rank, world)
        wl = full.shard(lo, hi)
        gm = gpu_model("student-35-1", "fp16", max_tokens=16384, max_sents=2048, workspaces=2)
        d_out = torch.zeros(wl.n, gm.Tmax, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(wl.n, dtype=torch.int32, device="cuda")
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            gm.translate_device(torch.from_numpy(wl.ids).cuda(), wl.off, d_out, d_len, caps=wl.caps,
                                workers=2)
        torch.cuda.synchronize()
        res = gather_device_outputs(d_out.cpu(), d_len.cpu())
        q.put((rank, None if res is None else (outputs_digest(*res), res[1].tolist())))
    finally:
        dist.destroy_process_group()


def test_whole_set_two_ranks_byte_identical():
    from synth import newstest_like
    from gpu_common import gpu_model
    from paper_2109_08008_b200.dist import outputs_digest
    full = newstest_like(N, 32000, start=40000)
    gm = gpu_model("student-35-1", "fp16", max_tokens=16384, max_sents=2048)
    d_out = torch.zeros(N, gm.Tmax, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(N, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        gm.translate_device(torch.from_numpy(full.ids).cuda(), full.off, d_out, d_len, caps=full.caps)
    torch.cuda.synchronize()
    lens = d_len.cpu().numpy()
    keep = np.arange(gm.Tmax)[None, :] < lens[:, None]
    ref = outputs_digest(d_out.cpu().numpy()[keep], lens)
    del gm
    torch.cuda.empty_cache()
    world, port = 2, 31500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    digest, merged_lens = got[0]
    assert merged_lens == lens.tolist()
    assert digest == ref
