"""Pins for oracle/batching.py: SPEC/hand-simulated examples + invariants."""
import os

import numpy as np

from oracle.batching import plan_batches, restore_order

GOLD = os.path.join(os.path.dirname(__file__), "golden", "plan_batches.txt")


def test_plan_golden():
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if not line:
            continue
        lens, tok, cap, exp = [p.strip() for p in line.split("|")]
        lens = [int(x) for x in lens.split(",")]
        got = plan_batches(lens, int(tok), int(cap))
        got_l = [[lens[i] for i in b] for b in got]
        exp_l = [[int(x) for x in grp.split(",")] for grp in exp.split(";")]
        assert got_l == exp_l, line


def test_plan_invariants():
    r = np.random.default_rng(0)
    for _ in range(50):
        lens = r.integers(1, 121, size=r.integers(1, 400))
        tok, cap = int(r.integers(120, 5000)), int(r.integers(1, 600))
        bs = plan_batches(lens, tok, cap)
        flat = [i for b in bs for i in b]
        assert sorted(flat) == list(range(len(lens)))        # each index exactly once
        for b in bs:
            assert len(b) <= cap
            assert len(b) == 1 or len(b) * lens[b[0]] <= tok   # token budget over padded length
            assert all(lens[b[0]] >= lens[i] for i in b)       # first is the longest
        seq = [(-int(lens[i]), i) for i in flat]
        assert seq == sorted(seq)                              # stable descending order


def test_restore_order_roundtrip():
    lens = [3, 9, 1, 9, 4]
    bs = plan_batches(lens, 10, 2)
    outs = [[f"s{i}" for i in b] for b in bs]
    assert restore_order(bs, outs, 5) == [f"s{i}" for i in range(5)]
