#!/usr/bin/env python
"""§8(f) rows f1/f2 measurement (GPU box): the paper's four-teacher ensemble (Table 1,
PAPER.md:40-44: 35-6, 35-6+DLCL, 40-6, 40-6+DLCL; random-init weights of that
architecture, FP16) decoding a newstest-shaped chunk with beam 4, as 1-best and as the
4-best lists of sequence-level KD.  Also the single 40-6+DLCL teacher for
the ensemble's cost ratio.  Prints one JSON object (target tokens/s, wall clock around a
synchronised call; the first call is a warm-up).

Usage: python tools/bench_ensemble.py [--n 512] [--max-tokens 4096] [--max-sents 128] [--eager]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import PRESETS, generate_weights, newstest_like  # noqa: E402
from paper_2109_08008_b200 import Model, Ensemble  # noqa: E402


def timed(fn, reps=1):
    fn()                      # warm-up (tensor maps, kernel attributes)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t0) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--max-tokens", type=int, default=4096)
    ap.add_argument("--max-sents", type=int, default=128)
    ap.add_argument("--eager", action="store_true",
                    help="legacy default stream: eager launches (no CUDA-graph decode steps)")
    a = ap.parse_args()
    if not a.eager:   # decode steps are captured and replayed as CUDA graphs off stream 0
        torch.cuda.set_stream(torch.cuda.Stream())
    names = ["ens-35-6", "ens-35-6-dlcl", "ens-40-6", "ens-40-6-dlcl"]
    lim = dict(max_tokens=a.max_tokens, max_sents=a.max_sents, max_tgt_len=200, beam=4)
    models = [Model(PRESETS[n], generate_weights(PRESETS[n], seed=3000 + i), precision="fp16", **lim)
              for i, n in enumerate(names)]
    wl = newstest_like(a.n, 32000, start=500_000)
    res = {"workload": f"{a.n} newstest-shaped sentences, batches {a.max_tokens} tokens / "
                       f"{a.max_sents} sentences, beam 4, FP16, random-init teachers, "
                       f"{'eager launches' if a.eager else 'CUDA-graph decode steps'}",
           "members": names}
    single = Ensemble([models[3]])
    (h, s, st), dt = timed(lambda: single.translate(wl.ids, wl.off, beam=4, caps=wl.caps))
    res["single_40_6_dlcl"] = {"tok_s": st["gen_tokens"] / dt, "s": dt, "gen_tokens": st["gen_tokens"]}
    ens = Ensemble(models)
    (h, s, st), dt = timed(lambda: ens.translate(wl.ids, wl.off, beam=4, caps=wl.caps))
    res["ensemble_1best"] = {"tok_s": st["gen_tokens"] / dt, "s": dt, "gen_tokens": st["gen_tokens"],
                             "decode_steps": st["decode_steps"]}
    (h, s, st), dt = timed(lambda: ens.translate(wl.ids, wl.off, beam=4, nbest=4, caps=wl.caps))
    res["ensemble_4best"] = {"tok_s": st["gen_tokens"] / dt, "s": dt, "gen_tokens": st["gen_tokens"],
                             "hypotheses": int(sum(len([x for x in hs if x]) for hs in h)),
                             "mean_best_score": float(np.mean([sc[0] for sc in s]))}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
