#!/usr/bin/env python
"""Time the library GEMMs (tcgen05 FP16) on the encoder / decoder shapes of the 35-1 model
with CUDA events (warm, inputs L2-resident or not as noted) and print TFLOP/s.
Usage (GPU box): python tools/gemm_bench.py [--tokens 16384] [--rows 256]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_08008_b200 import dev_gemm, dev_gemm_decode, dev_gemm_argmax  # noqa: E402


def bench(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--rows", type=int, default=256)
    a = ap.parse_args()
    d, F, V = 512, 2048, 32000
    g = torch.Generator(device="cuda").manual_seed(0)
    res = {}
    N = a.tokens
    for name, (M, Nn, K, resid, relu) in {
        "enc_qkv": (N, 3 * d, d, False, False), "enc_out": (N, d, d, True, False),
        "enc_ffn1": (N, F, d, False, True), "enc_ffn2": (N, d, F, True, False),
        "cross_kv": (N, 2 * d, d, False, False)}.items():
        A = torch.randn(M, K, device="cuda", generator=g).half()
        B = (torch.randn(Nn, K, device="cuda", generator=g) / K ** 0.5).half()
        bias = torch.zeros(Nn, device="cuda").half()
        R = torch.randn(M, Nn, device="cuda", generator=g).half() if resid else None
        C = torch.empty(M, Nn, device="cuda").half()
        ms = bench(lambda: dev_gemm(A, B, bias, R, relu=relu, out=C))
        ref = bench(lambda: torch.nn.functional.linear(A, B))     # cuBLAS, plain GEMM (context)
        res[name] = {"M": M, "N": Nn, "K": K, "us": ms * 1e3, "tflops": 2 * M * Nn * K / ms / 1e9,
                     "cublas_us": ref * 1e3}
    M = a.rows
    for name, (Nn, K, resid, relu) in {
        "dec_qkv": (3 * d, d, False, False), "dec_out": (d, d, True, False),
        "dec_ffn1": (F, d, False, True), "dec_ffn2": (d, F, True, False)}.items():
        A = torch.randn(M, K, device="cuda", generator=g).half()
        B = (torch.randn(Nn, K, device="cuda", generator=g) / K ** 0.5).half()
        bias = torch.zeros(Nn, device="cuda").half()
        R = torch.randn(M, Nn, device="cuda", generator=g).half() if resid else None
        C = torch.empty(M, Nn, device="cuda").half()
        ms = bench(lambda: dev_gemm_decode(A, B, bias, R, relu=relu, out=C), iters=100)
        byts = (Nn * K + M * K + M * Nn * (2 if resid else 1)) * 2
        res[name] = {"M": M, "N": Nn, "K": K, "us": ms * 1e3, "GBps": byts / ms / 1e6}
    A = torch.randn(M, d, device="cuda", generator=g).half()
    E = (torch.randn(V, d, device="cuda", generator=g) / d ** 0.5).half()
    ms = bench(lambda: dev_gemm_argmax(A, E), iters=100)
    res["vocab_argmax"] = {"M": M, "N": V, "K": d, "us": ms * 1e3, "GBps": V * d * 2 / ms / 1e6}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
