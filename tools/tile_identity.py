#!/usr/bin/env python
"""Are decode-GEMM results independent of the output tile shape?  Runs the 35-1 decoder
projections (seeded inputs) through nmt_dev_gemm_decode in child processes with
NMT_DEC_TILE = 64 / 128 / 256 (non-split) and compares the outputs bit for bit; then the
library's own policy ("auto": FFN2 split-K 2 in the cluster kernel up to 2048 rows, in
persistent KS = 2 units above) against the cluster kernel forced at every row count
(NMT_DEC_SPLITS = 2).
Usage (GPU box): python tools/tile_identity.py [rows ...]"""
import hashlib
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(rows):
    import torch
    from paper_2109_08008_b200 import dev_gemm_decode
    d, F = 512, 2048
    shapes = {"qkv": (3 * d, d, False, False), "self_out": (d, d, True, False),
              "ffn1": (F, d, False, True), "ffn2": (d, F, True, False)}
    for M in rows:
        g = torch.Generator(device="cuda").manual_seed(M)
        for name, (N, K, resid, relu) in shapes.items():
            A = torch.randn(M, K, device="cuda", generator=g).half()
            B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
            bias = torch.randn(N, device="cuda", generator=g).half()
            R = torch.randn(M, N, device="cuda", generator=g).half() if resid else None
            C = torch.empty(M, N, device="cuda").half()
            dev_gemm_decode(A, B, bias, R, relu=relu, out=C)
            torch.cuda.synchronize()
            print(f"{M} {name} {hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()}", flush=True)


def main():
    if sys.argv[1:2] == ["--child"]:
        child([int(x) for x in sys.argv[2:]])
        return
    rows = sys.argv[1:] or ["100", "1000", "4000"]
    res = {}
    for tile in ("64", "128", "256"):
        env = dict(os.environ, NMT_DEC_TILE=tile)
        r = subprocess.run([sys.executable, __file__, "--child"] + rows, env=env, capture_output=True, text=True)
        res[tile] = dict((" ".join(l.split()[:2]), l.split()[2]) for l in r.stdout.splitlines() if l.strip())
        if r.returncode:
            print(tile, r.stderr[-1500:])
    keys = sorted(res["64"])
    for k in keys:
        h = [res[t].get(k) for t in ("64", "128", "256")]
        print(k, "IDENTICAL" if len(set(h)) == 1 else "DIFFER", h)
    split = {}
    for mode, extra in (("auto", {}), ("cluster", {"NMT_DEC_SPLITS": "2"})):
        env = dict(os.environ, **extra)
        env.pop("NMT_DEC_TILE", None)
        r = subprocess.run([sys.executable, __file__, "--child"] + rows, env=env, capture_output=True, text=True)
        split[mode] = dict((" ".join(l.split()[:2]), l.split()[2]) for l in r.stdout.splitlines() if l.strip())
        if r.returncode:
            print(mode, r.stderr[-1500:])
    for k in sorted(split["auto"]):
        if k.endswith("ffn2"):
            h = [split["auto"].get(k), split["cluster"].get(k)]
            print(k, "split-K auto vs cluster:", "IDENTICAL" if len(set(h)) == 1 else "DIFFER", h)


if __name__ == "__main__":
    main()
