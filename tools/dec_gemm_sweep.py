#!/usr/bin/env python
"""Decode-step GEMM timing (GPU box): the six decoder-layer projections of the 35-1 model at
several live-row counts, launched back to back inside a CUDA graph (as in the decode step)
and timed by replaying the graph with CUDA events.  The configuration comes from the
library's decode policy, or NMT_DEC_TILE / NMT_DEC_SPLITS for tuning experiments.
Usage: python tools/dec_gemm_sweep.py [--rows 256,1024,2048]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_08008_b200 import dev_gemm_decode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", default="256,1024,2048")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    d, F = 512, 2048
    shapes = {"qkv": (3 * d, d, False, False), "self_out": (d, d, True, False),
              "cross_q": (d, d, False, False), "cross_out": (d, d, True, False),
              "ffn1": (F, d, False, True), "ffn2": (d, F, True, False)}
    g = torch.Generator(device="cuda").manual_seed(0)
    out = {}
    for M in [int(x) for x in a.rows.split(",")]:
        ops = []
        for name, (N, K, resid, relu) in shapes.items():
            A = torch.randn(M, K, device="cuda", generator=g).half()
            B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
            bias = torch.zeros(N, device="cuda").half()
            R = torch.randn(M, N, device="cuda", generator=g).half() if resid else None
            C = torch.empty(M, N, device="cuda").half()
            ops.append((name, A, B, bias, R, C, relu))
        s = torch.cuda.Stream()
        res = {}
        for name in [o[0] for o in ops] + ["all"]:
            todo = ops if name == "all" else [o for o in ops if o[0] == name]
            with torch.cuda.stream(s):
                for o in todo:   # warm (tensor maps, attributes)
                    dev_gemm_decode(o[1], o[2], o[3], o[4], relu=o[6], out=o[5])
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=s):
                for _ in range(a.reps):
                    for o in todo:
                        dev_gemm_decode(o[1], o[2], o[3], o[4], relu=o[6], out=o[5])
            graph.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                graph.replay()
            e1.record()
            torch.cuda.synchronize()
            res[name] = round(e0.elapsed_time(e1) / (5 * a.reps) * 1e3, 2)
        out[M] = res
    print(json.dumps({"cfg": {"tile": os.environ.get("NMT_DEC_TILE", "auto"),
                              "splits": os.environ.get("NMT_DEC_SPLITS", "auto")}, "us": out}))


if __name__ == "__main__":
    main()
