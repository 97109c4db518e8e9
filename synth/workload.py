"""Synthetic translation workloads (seeded input generator; no method arithmetic).

PAPER.md gives no length statistics: only 2998 sentences for newstest2018
(PAPER.md:70), 1M sentences for the task and caps of 120 source /
200 target tokens.  The recipe below is DESIGN.md's input
recipe:

  * DATA_SEED = 20200710, NumPy PCG64.
  * source length incl. EOS: n_i = clip(round(exp(N(ln 23, 0.6^2))), 2, 120)
  * per-sentence target cap: cap_i = clip(round(n_i * exp(N(ln 1.1, 0.15^2))), 2, 200)
  * ids: uniform in [4, V) for the first n_i - 1 positions, then EOS.

Every prefix of the 1M-sentence set is reproducible without generating the
rest of the ids (lengths come from one stream, ids from another).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import EOS_ID

DATA_SEED = 20200710
FULL_SET = 1_000_000


@dataclass
class Workload:
    ids: np.ndarray      # int32 [sum n_i] concatenated source ids (EOS-terminated)
    off: np.ndarray      # int64 [n+1] offsets into ids
    caps: np.ndarray     # int32 [n] per-sentence target caps (generated tokens)

    @property
    def n(self) -> int:
        return len(self.caps)

    def sentence(self, i: int) -> np.ndarray:
        return self.ids[self.off[i]:self.off[i + 1]]

    def lengths(self) -> np.ndarray:
        return np.diff(self.off).astype(np.int32)

    def shard(self, lo: int, hi: int) -> "Workload":
        o = self.off
        return Workload(self.ids[o[lo]:o[hi]].copy(), (o[lo:hi + 1] - o[lo]).astype(np.int64),
                        self.caps[lo:hi].copy())


def newstest_like(n: int, vocab: int, seed: int = DATA_SEED, start: int = 0,
                  full: int = FULL_SET, max_src: int = 120, max_tgt: int = 200) -> Workload:
    """Sentences [start, start+n) of the synthetic ``full``-sentence set."""
    assert 0 <= start and start + n <= full
    rl = np.random.Generator(np.random.PCG64(seed))
    lens = np.clip(np.rint(np.exp(rl.normal(np.log(23.0), 0.6, size=full))), 2, max_src).astype(np.int64)
    ratio = np.exp(rl.normal(np.log(1.1), 0.15, size=full))
    caps = np.clip(np.rint(lens * ratio), 2, max_tgt).astype(np.int32)
    body = lens - 1
    ri = np.random.Generator(np.random.PCG64(seed + 1))
    pre = int(body[:start].sum())
    cnt = int(body[start:start + n].sum())
    flat = ri.integers(4, vocab, size=pre + cnt, dtype=np.int64)[pre:].astype(np.int32)
    ln = lens[start:start + n]
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(ln, out=off[1:])
    ids = np.empty(int(off[-1]), dtype=np.int32)
    # place bodies and the terminating EOS (vectorised scatter)
    pos_eos = off[1:] - 1
    mask = np.ones(len(ids), dtype=bool)
    mask[pos_eos] = False
    ids[mask] = flat
    ids[pos_eos] = EOS_ID
    return Workload(ids, off, caps[start:start + n].copy())


def tiny_workload(n: int = 8, vocab: int = 1000, seed: int = 7, max_len: int = 16,
                  max_cap: int = 24) -> Workload:
    """C1: n sentences with n_i ~ U{2..max_len}, caps ~ U{1..max_cap}."""
    r = np.random.Generator(np.random.PCG64(seed))
    lens = r.integers(2, max_len + 1, size=n)
    caps = r.integers(1, max_cap + 1, size=n).astype(np.int32)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    ids = np.empty(int(off[-1]), dtype=np.int32)
    for i in range(n):
        ids[off[i]:off[i + 1] - 1] = r.integers(4, vocab, size=lens[i] - 1)
        ids[off[i + 1] - 1] = EOS_ID
    return Workload(ids, off, caps)


def random_tokens(n_rows: int, n_steps: int, vocab: int, seed: int = 11) -> np.ndarray:
    """Random forced target prefixes [n_rows, n_steps] in [4, V) (teacher forcing)."""
    r = np.random.Generator(np.random.PCG64(seed))
    return r.integers(4, vocab, size=(n_rows, n_steps)).astype(np.int32)
