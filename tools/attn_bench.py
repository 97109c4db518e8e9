#!/usr/bin/env python
"""Encoder attention micro-benchmark through nmt_dev_attn_encoder (FP16, d = 512, 8 heads,
RPR k = 8): one 32768-token batch per padded length S, lengths drawn like the bench
workload (every sentence of a batch within the length class, sorted).  CUDA-event time per
launch (median of 5 samples of 20 back-to-back launches), effective HBM GB/s of the algorithmic bytes
(read Q/K/V of B*S rows, write B*S output rows).  NMT_ENC_ATTN=0 selects the previous
kernel for A/B.  Usage: python tools/attn_bench.py [S ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_08008_b200 import dev_attn_encoder  # noqa: E402


def main():
    d, H, kc = 512, 8, 8
    rng = np.random.default_rng(0)
    relk = torch.randn(2 * kc + 1, d // H, dtype=torch.float16, device="cuda") * 0.5
    relv = torch.randn(2 * kc + 1, d // H, dtype=torch.float16, device="cuda") * 0.5
    sizes = [int(x) for x in sys.argv[1:]] or [12, 16, 24, 32, 40, 48, 64, 96, 120]
    for S in sizes:
        B = 32768 // S
        qkv = torch.randn(B * S, 3 * d, dtype=torch.float16, device="cuda")
        lens = np.clip(rng.integers(max(2, S - 8), S + 1, size=B), 2, S)
        lens[0] = S
        ln = torch.from_numpy(np.sort(lens)[::-1].copy().astype(np.int32)).cuda()
        for _ in range(3):
            dev_attn_encoder(qkv, ln, relk, relv, B, S, H, kc)
        ts = []
        for _ in range(5):   # 20 back-to-back launches per sample: host call overhead hidden
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                dev_attn_encoder(qkv, ln, relk, relv, B, S, H, kc)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20)
        ms = float(np.median(ts))
        byts = B * S * 4 * d * 2
        print(f"S={S:4d} B={B:5d} {1000 * ms:8.1f} us  {byts / ms / 1e6:7.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
