"""Shared helpers for the -m gpu parity tests (CUDA path vs oracle on identical inputs)."""
from __future__ import annotations

import functools

import numpy as np

from synth import PRESETS, generate_weights

# Tolerances (BASELINE.json north_star): FP32 mode 1e-4 relative to max(1, |row|_inf),
# FP16 mode 2e-2 absolute per logit.
TOL = {"fp32": 1e-4, "fp16": 2e-2}
# A position is margin-safe when the oracle's top1 - top2 logit gap exceeds 2 tol (SURVEY
# §8(c): 4e-2 in FP16, 2e-4 * max(1, max|logit|) in FP32); only there is the GPU argmax pinned.


def safe_gap(prec: str, scale: float = 1.0) -> float:
    return 2 * TOL[prec] * (max(1.0, scale) if prec == "fp32" else 1.0)


def safe_prefix_len(gaps, scales, prec: str) -> int:
    """Number of leading generated positions that are margin-safe (oracle log)."""
    k = 0
    while k < len(gaps) and gaps[k] > safe_gap(prec, scales[k]):
        k += 1
    return k


@functools.lru_cache(maxsize=None)
def weights(name: str, eos_boost: float = 1.0, **over):
    cfg = PRESETS[name].replace(**over) if over else PRESETS[name]
    return cfg, generate_weights(cfg, eos_boost=eos_boost)


@functools.lru_cache(maxsize=None)
def oracle_model(name: str, eos_boost: float = 1.0):
    from oracle import OracleModel
    cfg, W = weights(name, eos_boost)
    return OracleModel(W, cfg)


def gpu_model(name: str, prec: str, eos_boost: float = 1.0, **lim):
    from paper_2109_08008_b200 import Model
    cfg, W = weights(name, eos_boost)
    return Model(cfg, W, precision=prec, **lim)


def logits_close(g: np.ndarray, o: np.ndarray, prec: str):
    """Row-wise check; returns (ok, worst excess ratio)."""
    if prec == "fp32":
        scale = np.maximum(1.0, np.abs(o).max(axis=-1, keepdims=True))
        err = np.abs(g - o) / scale
    else:
        err = np.abs(g - o)
    worst = float(err.max()) if err.size else 0.0
    return worst <= TOL[prec], worst


def margin_safe(o_logits: np.ndarray, prec: str) -> np.ndarray:
    top2 = np.partition(o_logits, -2, axis=-1)[..., -2:]
    gap = top2[..., 1] - top2[..., 0]
    tol = TOL[prec] * (np.maximum(1.0, np.abs(o_logits).max(axis=-1)) if prec == "fp32" else 1.0)
    return gap > 2 * tol


def pad_batch(srcs):
    B = len(srcs)
    S = max(len(s) for s in srcs)
    a = np.zeros((B, S), dtype=np.int32)
    for i, s in enumerate(srcs):
        a[i, :len(s)] = s
    return a, np.array([len(s) for s in srcs], dtype=np.int32)


def _step_fn(om, src):
    """Cached oracle decoder for one sentence: returns f(prev_token, t) -> FP64 logits."""
    enc, sl = om.encode_batch([list(src)])
    ckv = om.cross_kv(enc)
    cache = om.new_cache(1, om.cfg.max_tgt_len + 1)

    def f(prev, t):
        return om.decoder_step(np.array([prev]), t, cache, ckv, sl)[0]
    return f


def greedy_valid(om, src, cap, toks, prec: str):
    """Validity of a GPU greedy output where it leaves the oracle's (several correct results,
    SURVEY §8(c) A23): teacher-force the oracle along [BOS] + toks (+ EOS if the GPU stopped
    before the cap) and require every chosen token to be within 2 tol of the oracle's maximum
    logit at its step — the argmax under the FP16 (FP32) error bound.  Returns (ok, step)."""
    from synth import BOS_ID, EOS_ID
    cap = int(min(cap, om.cfg.max_tgt_len))
    if len(toks) > cap or EOS_ID in toks:
        return False, -1
    seq = list(toks) + ([EOS_ID] if len(toks) < cap else [])
    f = _step_fn(om, src)
    prev = BOS_ID
    for t, w in enumerate(seq):
        lo = f(prev, t)
        if lo[w] < lo.max() - safe_gap(prec, float(np.abs(lo).max())):
            return False, t
        prev = w
    return True, None


def seq_logprob(step_logprobs, toks, cap):
    """FP64 oracle score (sum of log-probabilities, R16) of a finished hypothesis: its tokens
    and the terminating EOS when it ended before the cap.  step_logprobs(prefixes) -> list of
    log-probability vectors (oracle.search conventions)."""
    from synth import BOS_ID, EOS_ID
    seq = list(toks) + ([EOS_ID] if len(toks) < cap else [])
    pre = [BOS_ID]
    sc = 0.0
    for w in seq:
        sc += float(step_logprobs([pre])[0][w])
        pre = pre + [w]
    return sc


def oracle_step_logprobs(om, src):
    from oracle.search import prefix_logprobs
    enc, sl = om.encode_batch([list(src)])
    ckv = om.cross_kv(enc)
    return lambda prefixes: prefix_logprobs(om, ckv, sl, prefixes)


def beam_valid(step_logprobs, cap, got, ref, got_score=None, prec="fp16"):
    """FP16 beam acceptance (several correct results): equal to the oracle's hypothesis, or
    within the FP16 error bound of it — every log-probability carries <= 2 tol of error (logit
    + log-sum-exp), so a hypothesis of T tokens <= 2 tol T, and two compared scores 4 tol T.
    The GPU hypothesis is valid if its FP64 oracle score is within 4 tol T of the oracle's
    beam result, and (when given) the GPU's own score within 2 tol T of that FP64 score."""
    cap = int(cap)
    if list(got) == list(ref) and got_score is None:
        return True
    T = max(len(got), len(ref)) + 1
    s_got = seq_logprob(step_logprobs, got, cap)
    ok = True
    if list(got) != list(ref):
        s_ref = seq_logprob(step_logprobs, ref, cap)
        ok = s_got >= s_ref - 4 * TOL[prec] * T
    if got_score is not None:
        ok = ok and abs(got_score - s_got) <= 2 * TOL[prec] * T
    return ok
