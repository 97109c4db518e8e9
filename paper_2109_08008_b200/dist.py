"""Multi-GPU plumbing (host side only): sentence sharding, max-over-ranks timing and the
end-of-run gather of outputs — the paper's "split the input into several parts ... merge
each part of translations to one file in the original order", with one
process per B200 instead of one per CPU core.

No collective sits on the data path: ranks translate disjoint sentence ranges
independently; torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only for
barriers, the timing/count reductions and the final gather.
"""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of n sentences for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def chunk_index(step: int, rank: int, world: int) -> int:
    """Weak-scaling bench: step k of rank r translates global chunk k*world + r (disjoint)."""
    return step * world + rank


def reduce_timing(ms: float, tokens: float, device=None):
    """(max over ranks of ms, sum over ranks of tokens); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ms, tokens
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([tokens], dtype=torch.float64, device=device)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return t.item(), c.item()


def gather_outputs(outs: list, device=None):
    """Gather every rank's per-sentence token lists to rank 0 in rank order (= original
    order for contiguous shards).  Returns the merged list on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(outs)
    world, rank = dist.get_world_size(), dist.get_rank()
    lens = np.array([len(o) for o in outs], dtype=np.int64)
    flat = np.concatenate([np.asarray(o, dtype=np.int32) for o in outs]) if outs else np.zeros(0, np.int32)
    meta = torch.tensor([len(outs), len(flat)], dtype=torch.int64, device=device)
    metas = [torch.zeros(2, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(metas, meta)
    n_max = int(max(m[0] for m in metas))
    t_max = int(max(m[1] for m in metas))
    pad_l = torch.zeros(n_max, dtype=torch.int64, device=device)
    pad_l[:len(lens)] = torch.from_numpy(lens)
    pad_t = torch.zeros(max(t_max, 1), dtype=torch.int32, device=device)
    pad_t[:len(flat)] = torch.from_numpy(flat)
    all_l = [torch.zeros_like(pad_l) for _ in range(world)]
    all_t = [torch.zeros_like(pad_t) for _ in range(world)]
    dist.all_gather(all_l, pad_l)
    dist.all_gather(all_t, pad_t)
    if rank != 0:
        return None
    merged = []
    for r in range(world):
        n_r = int(metas[r][0])
        ls = all_l[r][:n_r].cpu().numpy()
        toks = all_t[r].cpu().numpy()
        off = 0
        for L in ls:
            merged.append(toks[off:off + L].tolist())
            off += L
    return merged


def gather_device_outputs(d_out, d_len, device=None):
    """Whole-set merge (C5, "merge ... in the original order"): every rank
    holds its contiguous shard's outputs as d_out [n_r][stride] int32 (EOS included when
    produced) and d_len [n_r]; the tokens are compacted on the rank's device, gathered with
    the process group's all_gather (NCCL on GPUs: padded to the largest shard) and
    concatenated in rank order on rank 0.  Returns (flat int32 tokens, lengths int32) as
    NumPy arrays on rank 0, None elsewhere; without a process group the local arrays."""
    import torch
    import torch.distributed as dist
    n_r, stride = d_out.shape
    dev = d_out.device if device is None else device
    lens = d_len.to(torch.int64)
    keep = torch.arange(stride, device=d_out.device)[None, :] < lens[:, None]
    flat = d_out[keep].to(torch.int32)            # row-major: sentence by sentence
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return flat.cpu().numpy(), d_len.to(torch.int32).cpu().numpy()
    world, rank = dist.get_world_size(), dist.get_rank()
    meta = torch.tensor([n_r, flat.numel()], dtype=torch.int64, device=dev)
    metas = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(metas, meta)
    n_max = int(max(int(m[0]) for m in metas))
    t_max = max(1, int(max(int(m[1]) for m in metas)))
    pl = torch.zeros(n_max, dtype=torch.int32, device=dev)
    pl[:n_r] = d_len.to(torch.int32).to(dev)
    pt = torch.zeros(t_max, dtype=torch.int32, device=dev)
    pt[:flat.numel()] = flat.to(dev)
    al = [torch.zeros_like(pl) for _ in range(world)]
    at = [torch.zeros_like(pt) for _ in range(world)]
    dist.all_gather(al, pl)
    dist.all_gather(at, pt)
    if rank != 0:
        return None
    toks = [at[r][:int(metas[r][1])].cpu().numpy() for r in range(world)]
    ls = [al[r][:int(metas[r][0])].cpu().numpy() for r in range(world)]
    return np.concatenate(toks).astype(np.int32), np.concatenate(ls).astype(np.int32)


def outputs_digest(flat: np.ndarray, lens: np.ndarray) -> str:
    """SHA-256 over (lengths, tokens) little-endian int32: byte-identical merged outputs
    across world sizes have equal digests (SURVEY §8(e) check)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(lens, dtype="<i4").tobytes())
    h.update(np.ascontiguousarray(flat, dtype="<i4").tobytes())
    return h.hexdigest()
