#!/usr/bin/env python
"""A/B of the decode step (one worker, profile mode 3: each step's CUDA graph between two
event nodes): unfused vs fused (and NMT_FUSE_ROWS variants) at the paper budget (4096 /
512) and the bench budget (65536 / 8192), plus whole-chunk tok/s with the bench's 4 workers.

Usage (GPU box): python tools/step_ab.py [sentences] [modes...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
BUCKETS = [(1, 16), (17, 64), (65, 148), (149, 512), (513, 1024), (1025, 2048), (2049, 8192)]


def child(mode_env, n):
    import numpy as np
    import torch
    from synth import PRESETS, generate_weights, newstest_like
    from paper_2109_08008_b200 import Model
    cfg = PRESETS["student-35-1"]
    W = generate_weights(cfg)
    wl = newstest_like(n, cfg.vocab_size, start=0)
    big = newstest_like(96000, cfg.vocab_size, start=96000)
    out = {}
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    d_out = torch.empty(96000, 200, dtype=torch.int32, device="cuda")
    d_len = torch.empty(96000, dtype=torch.int32, device="cuda")
    for mt, ms in ((4096, 512), (65536, 8192)):
        m = Model(cfg, W, precision="fp16", max_tokens=mt, max_sents=ms, workspaces=4)
        ids = torch.from_numpy(wl.ids).cuda()
        m.translate_device(ids, wl.off, d_out, d_len, caps=wl.caps)          # warm graphs
        m.profile(3)
        m.translate_device(ids, wl.off, d_out, d_len, caps=wl.caps)
        rec = m.profile_steps()
        m.profile(0)
        b = {}
        for lo, hi in BUCKETS:
            v = sorted(ms_ for t, live, ms_ in rec if lo <= live <= hi and 12 <= t <= 20)
            if v:
                b[f"{lo}-{hi}"] = round(v[len(v) // 2] * 1e3, 1)
        mean = sum(x for _, _, x in rec) / len(rec) * 1e3
        # whole chunk, 4 workers, device-resident
        bid = torch.from_numpy(big.ids).cuda()
        m.translate_device(bid, big.off, d_out, d_len, caps=big.caps, workers=4)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        st = m.translate_device(bid, big.off, d_out, d_len, caps=big.caps, workers=4)
        e1.record(s)
        torch.cuda.synchronize()
        out[f"{mt}/{ms}"] = {"step_us_median_by_live_rows": b, "step_us_mean": round(mean, 1),
                             "chunk_tok_s": round(st["gen_tokens"] / (e0.elapsed_time(e1) / 1e3))}
        del m
    print("RESULT " + json.dumps(out), flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(None, int(sys.argv[2]))
        return
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12000
    modes = sys.argv[2:] or ["unfused", "fused"]
    envs = {"unfused": {"NMT_NO_FUSE": "1"}, "fused": {}, "one": {"NMT_FUSE_ROWS": "100000"},
            "seg": {"NMT_FUSE_ROWS": "0"}, "f512": {"NMT_FUSE_ROWS": "512"},
            "f2048": {"NMT_FUSE_ROWS": "2048"}}
    res = {}
    for mode in modes:
        env = dict(os.environ)
        for k in ("NMT_NO_FUSE", "NMT_FUSE_ROWS"):
            env.pop(k, None)
        env.update(envs[mode])
        r = subprocess.run([sys.executable, __file__, "--child", str(n)], env=env, capture_output=True,
                           text=True)
        line = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        res[mode] = json.loads(line[-1][7:]) if line else {"error": r.stderr[-2000:]}
        print(mode, json.dumps(res[mode]), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
