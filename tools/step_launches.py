#!/usr/bin/env python
"""One graph-replayed decode step of the 35-1 model at a fixed live-row count (paper budget
rows), for an ncu launch list: python tools/step_launches.py [rows] [t] — run under
ncu --metrics gpu__time_duration.sum (the last 12 launches are the measured step)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from synth import PRESETS, generate_weights, random_tokens
    from paper_2109_08008_b200 import Model
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 148
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    cfg = PRESETS["student-35-1"]
    m = Model(cfg, generate_weights(cfg), precision="fp16", max_tokens=4096 * 4, max_sents=512)
    S = 28
    src = random_tokens(rows, S, cfg.vocab_size, seed=5).astype(np.int32)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = m.encode(torch.from_numpy(src).cuda(), [S] * rows, tgt_cap=[200] * rows)
        for t in range(T):
            b.decode_step(n_live=rows)
            b.prune(ratio=-1.0, want_map=False)
    torch.cuda.synchronize()
    print("done", rows, T)


if __name__ == "__main__":
    main()
