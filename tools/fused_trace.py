#!/usr/bin/env python
"""Timeline of one fused decode-step launch (csrc/decode_fused.cu, NMT_FUSED_TRACE): per
phase the first receive / last completion relative to the kernel's first CTA start, and the
median item wait (received -> inputs ready) and work (ready -> done) times, in us.

Usage (GPU box): python tools/fused_trace.py [rows ...]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NMT_FUSED_TRACE"] = "1"
os.environ.setdefault("NMT_FUSE_ROWS", "100000")

PH = ["embed+LN", "QKV", "self-attn", "self-out", "cross-q", "cross-attn", "cross-out", "FFN1",
      "FFN2", "final LN"]


def main():
    import numpy as np
    import torch
    from synth import PRESETS, generate_weights, newstest_like
    from paper_2109_08008_b200 import Model
    from paper_2109_08008_b200.nmt import lib, _check
    cfg = PRESETS["student-35-1"]
    W = generate_weights(cfg)
    for R in [int(x) for x in sys.argv[1:]] or [148, 1024]:
        m = Model(cfg, W, precision="fp16", max_tokens=max(4096, R * 128), max_sents=max(512, R))
        wl = newstest_like(R, 32000, start=100)
        L = wl.lengths()
        S = int(L.max())
        src = np.zeros((R, S), dtype=np.int32)
        for i in range(R):
            src[i, :L[i]] = wl.sentence(i)
        b = m.encode(torch.from_numpy(src).cuda(), L)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for t in range(16):
            if t == 15:
                ev[0].record()
            b.decode_step(n_live=R)
            if t == 15:
                ev[1].record()
            b.prune(ratio=-1.0, want_map=False)
        torch.cuda.synchronize()
        buf = (C.c_uint64 * (4 * 65536 + 1024))()
        _check(lib().nmt_debug_fused_trace(m.h, buf, len(buf)))
        a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64)
        starts = a[4 * 65536:4 * 65536 + 148]
        starts = starts[starts > 0]
        t0 = starts.min()
        rec = a[:4 * 65536].reshape(-1, 4)
        rec = rec[rec[:, 3] > 0]
        ph = rec[:, 0] >> 40
        print(f"R = {R}: decode_step (fused + vocab + finish) {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us; "
              f"CTA start spread {(starts.max() - t0) / 1e3:.1f} us; items {len(rec)}")
        print(f"  {'phase':12s} {'items':>5s} {'first_recv':>10s} {'last_done':>9s} {'med_wait':>8s} "
              f"{'med_work':>8s} {'max_work':>8s}")
        for p in range(10):
            r = rec[ph == p]
            if not len(r):
                continue
            print(f"  {PH[p]:12s} {len(r):5d} {(r[:, 1].min() - t0) / 1e3:10.1f} "
                  f"{(r[:, 3].max() - t0) / 1e3:9.1f} {np.median(r[:, 2] - r[:, 1]) / 1e3:8.1f} "
                  f"{np.median(r[:, 3] - r[:, 2]) / 1e3:8.1f} {(r[:, 3] - r[:, 2]).max() / 1e3:8.1f}")
        del b, m


if __name__ == "__main__":
    main()
