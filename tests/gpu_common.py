"""Shared helpers for the -m gpu parity tests (CUDA path vs oracle on identical inputs)."""
from __future__ import annotations

import functools

import numpy as np

from synth import PRESETS, generate_weights

# Tolerances (BASELINE.json north_star): FP32 mode 1e-4 relative to max(1, |row|_inf),
# FP16 mode 2e-2 absolute per logit.
TOL = {"fp32": 1e-4, "fp16": 2e-2}
# free-running comparisons stop at the first oracle top1-top2 gap below this
SAFE_GAP = {"fp32": 2e-3, "fp16": 4e-2}


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
