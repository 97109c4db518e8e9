"""ORACLE (test infrastructure only) — dynamic batching and order restoration.

* plan_batches: "a dynamic batching scheme that maximizes the number of
  sentences in the batch while limiting the number of tokens",
  "fixed batch size (number of sentences) of 512 on the GPU",
  inputs sorted "in descending order of length".  Reading R17:
  stable sort by (-len, index); b = min(max_sents, floor(max_tokens/len_first),
  remaining), at least 1.  Pinned: SPEC example [5,4,3,2] budget 10 ->
  [[5,4],[3,2]] (tests/golden/plan_batches.txt) + coverage/budget invariants.
* restore_order: "merge each part of translations ... in the original order"
  (PAPER.md:131).  Pinned: permutation round trip.
"""
from __future__ import annotations

import numpy as np


def plan_batches(lengths, max_tokens: int, max_sents: int):
    lengths = np.asarray(lengths)
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    batches = []
    i = 0
    while i < len(order):
        first = int(lengths[order[i]])
        b = min(max_sents, max(1, max_tokens // first), len(order) - i)
        batches.append(order[i:i + b])
        i += b
    return batches


def restore_order(batches, outputs_per_batch, n):
    out = [None] * n
    for idx, outs in zip(batches, outputs_per_batch):
        for i, o in zip(idx, outs):
            out[i] = o
    return out
