#!/usr/bin/env python
"""Per-class device time of decode steps at a fixed live-row count (35-1 FP16 greedy, step
API, eager launches with per-kernel events, no pruning): for each row count B and step
window [t0, t1), the mean us per step of every kernel class and its achieved bandwidth /
FLOP rate against the class's algorithmic bytes / FLOPs.

Usage (GPU box): python tools/dec_classes.py [B ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from synth import PRESETS, generate_weights, random_tokens
    from paper_2109_08008_b200 import Model
    cfg = PRESETS["student-35-1"]
    W = generate_weights(cfg)
    rows = [int(x) for x in sys.argv[1:]] or [148, 1024, 4096, 8192]
    windows = [(0, 8), (8, 24), (24, 56), (56, 120)]
    res = {}
    for B in rows:
        S = 30
        m = Model(cfg, W, precision="fp16", max_tokens=max(65536, B * S), max_sents=max(8192, B),
                  max_tgt_len=200)
        src = random_tokens(B, S, cfg.vocab_size, seed=B).astype(np.int32)
        b = m.encode(torch.from_numpy(src).cuda(), [S] * B, tgt_cap=[200] * B)
        out = {}
        t = 0
        for t0, t1 in windows:
            while t < t0:
                b.decode_step(n_live=B)
                b.prune(ratio=-1.0, want_map=False)
                t += 1
            torch.cuda.synchronize()
            m.profile(2)
            while t < t1:
                b.decode_step(n_live=B)
                b.prune(ratio=-1.0, want_map=False)
                t += 1
            prof = m.profile(-1)
            m.profile(0)
            n = t1 - t0
            out[f"{t0}-{t1}"] = {k: {"us": round(v["ms"] * 1e3 / n, 1),
                                     "GB/s": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] else 0,
                                     "TF/s": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 1) if v["ms"] else 0}
                                 for k, v in prof.items()}
            tot = sum(v["ms"] for v in prof.values()) * 1e3 / n
            out[f"{t0}-{t1}"]["total_us"] = round(tot, 1)
        res[B] = out
        print(B, json.dumps(out), flush=True)
        del b, m
    print("RESULT " + json.dumps(res))


if __name__ == "__main__":
    main()
