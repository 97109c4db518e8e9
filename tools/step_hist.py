#!/usr/bin/env python
"""Decode-step histogram (GPU box): translate a slice of the bench workload with step timing
(profile mode 3) and print step count / device time per live-row bucket, to see how much
decode time the low-occupancy tail steps take.  Usage: python tools/step_hist.py [n_sents]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import PRESETS, generate_weights, newstest_like  # noqa: E402
from paper_2109_08008_b200 import Model  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
    mt, ms = int(os.environ.get("MT", 65536)), int(os.environ.get("MS", 8192))
    cfg = PRESETS["student-35-1"]
    m = Model(cfg, generate_weights(cfg), precision="fp16", max_tokens=mt, max_sents=ms)
    wl = newstest_like(n, cfg.vocab_size, start=0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    d_ids = torch.from_numpy(wl.ids).cuda()
    d_out = torch.empty(n, m.Tmax, dtype=torch.int32, device="cuda")
    d_len = torch.empty(n, dtype=torch.int32, device="cuda")
    m.translate_device(d_ids, wl.off, d_out, d_len, caps=wl.caps, workers=1)   # warm
    m.profile(3)
    st = m.translate_device(d_ids, wl.off, d_out, d_len, caps=wl.caps, workers=1)
    rec = np.array(m.profile_steps(), dtype=np.float64)
    m.profile(0)
    live, ms_ = rec[:, 1], rec[:, 2]
    print(f"{st['batches']} batches, {len(rec)} steps, {ms_.sum():.1f} ms of decode steps, "
          f"{st['gen_tokens']} tokens")
    for lo, hi in [(1, 16), (17, 64), (65, 148), (149, 512), (513, 2048), (2049, 8192), (8193, 1 << 20)]:
        k = (live >= lo) & (live <= hi)
        if k.any():
            print(f"rows {lo:5d}-{hi:<7d} steps {k.sum():6d} ({100 * k.mean():5.1f} %)  "
                  f"time {ms_[k].sum():8.1f} ms ({100 * ms_[k].sum() / ms_.sum():5.1f} %)  "
                  f"mean {1e3 * ms_[k].mean():6.1f} us  rows*steps {int((live[k]).sum())}")


if __name__ == "__main__":
    main()
