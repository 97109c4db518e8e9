#!/usr/bin/env python
"""Timeline of one persistent tcgen05 GEMM launch (NMT_GEMM_TRACE): per unit, the mainloop
(MMA: accumulator free -> last commit), the epilogue of warp 4 (accumulator seen -> released
-> last store issued), the MMA's wait for a free accumulator and the epilogue's wait for a
full one — medians over the units of all CTAs, in us.

Usage (GPU box): python tools/gemm_trace.py [M] [N] [K] [residual 0/1] [relu 0/1]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NMT_GEMM_TRACE"] = "1"


def main():
    import numpy as np
    import torch
    from paper_2109_08008_b200 import dev_gemm
    from paper_2109_08008_b200.nmt import lib, _check
    M, N, K = [int(x) for x in (sys.argv[1:4] or [65520, 1536, 512])]
    resid = len(sys.argv) > 4 and sys.argv[4] == "1"
    relu = len(sys.argv) > 5 and sys.argv[5] == "1"
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda").half()
    R = torch.randn(M, N, device="cuda", generator=g).half() if resid else None
    Cc = torch.empty(M, N, device="cuda").half()
    for _ in range(3):
        dev_gemm(A, B, bias, R, relu=relu, out=Cc)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (148 * 32 * 8))()
    _check(lib().nmt_debug_gemm_trace(buf, len(buf)))
    a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(148, 32, 8)
    ok = (a > 0).all(axis=2)
    t0 = a[ok][:, 2].min()
    u = a[ok]
    d = lambda x, y: (u[:, y] - u[:, x]) / 1e3
    med = lambda v: float(np.median(v))
    # per CTA consecutive units: MMA wait for a free accumulator = stamp2(k) - stamp3(k-1)
    mw, ew = [], []
    for c in range(148):
        ks = [k for k in range(32) if ok[c, k]]
        for k in ks[1:]:
            mw.append((a[c, k, 2] - a[c, k - 1, 3]) / 1e3)
    print(f"GEMM {M}x{N}x{K} resid={int(resid)} relu={int(relu)}: units traced {len(u)}, "
          f"span {(u[:, 7].max() - t0) / 1e3:.1f} us")
    print(f"  mainloop (acc free -> last commit)      median {med(d(2, 3)):6.2f} us")
    print(f"  producer (first -> last load issued)    median {med(d(0, 1)):6.2f} us")
    print(f"  epilogue wait for acc (4 -> 5)          median {med(d(4, 5)):6.2f} us")
    print(f"  epilogue drain (acc seen -> released)   median {med(d(5, 6)):6.2f} us")
    print(f"  epilogue tail (released -> last store)  median {med(d(6, 7)):6.2f} us")
    print(f"  epilogue busy (acc seen -> last store)  median {med(d(5, 7)):6.2f} us")
    print(f"  MMA wait for a free accumulator         median {med(np.array(mw)) if mw else 0:6.2f} us")
    print(f"  commit -> epilogue sees acc (3 -> 5)    median {med(d(3, 5)):6.2f} us")


if __name__ == "__main__":
    main()
