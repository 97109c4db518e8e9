#!/usr/bin/env python
"""Per-tile timeline of the tcgen05 encoder attention (CTA 0): stamps relative to the first
Q/K TMA, in us.  Usage (GPU box): NMT_ENC_ATTN=2 NMT_ATTN_TRACE=1 python tools/attn_trace.py S"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_08008_b200 import dev_attn_encoder  # noqa: E402
from paper_2109_08008_b200.nmt import lib, _check  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 32
d, H, kc = 512, 8, 8
B = 32768 // S
qkv = torch.randn(B * S, 3 * d, dtype=torch.float16, device="cuda")
ln = torch.full((B,), S, dtype=torch.int32, device="cuda")
relk = torch.randn(17, 64, dtype=torch.float16, device="cuda") * 0.5
relv = torch.randn(17, 64, dtype=torch.float16, device="cuda") * 0.5
for _ in range(3):
    dev_attn_encoder(qkv, ln, relk, relv, B, S, H, kc)
buf = (C.c_uint64 * 1024)()
_check(lib().nmt_debug_attn_trace(buf, 1024))
a = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(64, 16)[:, :13]
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
print("tile  qkTMA  vTMA  QKiss  Sseen  Pready  PViss  Oseen  Tfree  qa_dn  p1_dn  p2_dn  bnd_dn fence_dn")
for k, r in enumerate(a[:20]):
    print(f"{k:4d} " + " ".join(f"{(x - t0) / 1e3:6.2f}" if x > 0 else "     -" for x in r))
