#!/usr/bin/env python
"""Tied vocab projection + argmax (nmt_dev_gemm_argmax, 35-1 shapes: N = 32000, K = 512) at
several row counts, CUDA-event timed; NMT_GEMM_DBG bits select the tuning variants (1 = drain
TMEM only, 32 = MMAs on stale tiles without operand TMA).
Usage (GPU box): python tools/vocab_bench.py [rows ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_08008_b200 import dev_gemm_argmax  # noqa: E402


def main():
    rows = [int(x) for x in sys.argv[1:]] or [148, 1024, 4096, 8192, 16384]
    V, d = 32000, 512
    g = torch.Generator(device="cuda").manual_seed(0)
    E = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5).half()
    out = {}
    for M in rows:
        A = torch.randn(M, d, device="cuda", generator=g).half()
        for _ in range(3):
            dev_gemm_argmax(A, E)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            dev_gemm_argmax(A, E)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / n * 1e3
        out[M] = {"us": round(us, 1), "TF/s": round(2 * M * V * d / us / 1e6, 1)}
    print(json.dumps({"dbg": os.environ.get("NMT_GEMM_DBG", "0"), "vocab_argmax": out}))


if __name__ == "__main__":
    main()
