"""Deterministic random-init weights (seeded input generator; no method arithmetic).

No trained weights exist for the paper's models (PAPER.md:33-34 trains with
fairseq on WMT data that is not available), so both the oracle and the CUDA
path consume the same synthetic weights, generated here once as
FP16-representable values (reading R6/R6b).

Generator: counter-based splitmix64,
    u(seed, tid, i) = (splitmix64(seed ^ (tid * 0x9E3779B97F4A7C15) + i) >> 11) * 2^-53
where ``tid`` is the tensor's index in the canonical name order.  Values are
``(2u - 1) * sqrt(3) * sigma`` rounded once to FP16 (so the FP16 and FP32 GPU
modes and the FP64 oracle see bit-identical weights).

Layout is nn.Linear's ``[out, in]`` for every projection.
"""
from __future__ import annotations

import math
from collections import OrderedDict

import numpy as np

from .config import ModelConfig, EOS_ID

WEIGHT_SEED = 2109
G_DEC = 32.0  # decoder sub-layer output gain (reading R6b)

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, tid: int, n: int) -> np.ndarray:
    """u in [0,1): 53-bit mantissa of splitmix64(seed ^ tid*GOLD + i), i = 0..n-1."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) ^ (np.uint64(tid) * _GOLD)
        x = base + np.arange(n, dtype=np.uint64)
    return (splitmix64(x) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def canonical_shapes(cfg: ModelConfig) -> "OrderedDict[str, tuple]":
    """Canonical tensor names -> shapes (SURVEY Appendix B naming)."""
    d, F, V = cfg.d_model, cfg.d_ffn, cfg.vocab_size
    R = 2 * cfg.max_rel_pos + 1
    dh = cfg.d_head
    s: "OrderedDict[str, tuple]" = OrderedDict()
    s["emb"] = (V, d)
    for l in range(cfg.enc_layers):
        p = f"enc.{l}."
        s[p + "attn_ln.g"] = (d,); s[p + "attn_ln.b"] = (d,)
        s[p + "qkv.w"] = (3 * d, d); s[p + "qkv.b"] = (3 * d,)
        s[p + "out.w"] = (d, d); s[p + "out.b"] = (d,)
        if cfg.use_rpr:
            s[p + "rel_k"] = (R, dh); s[p + "rel_v"] = (R, dh)
        s[p + "ffn_ln.g"] = (d,); s[p + "ffn_ln.b"] = (d,)
        s[p + "ffn1.w"] = (F, d); s[p + "ffn1.b"] = (F,)
        s[p + "ffn2.w"] = (d, F); s[p + "ffn2.b"] = (d,)
    if cfg.use_dlcl:
        for k in range(cfg.enc_layers + 1):
            s[f"enc.dlcl.ln.{k}.g"] = (d,); s[f"enc.dlcl.ln.{k}.b"] = (d,)
        L1 = cfg.enc_layers + 1
        s["enc.dlcl.w"] = (L1 * (L1 + 1) // 2,)  # rows m=1..L+1, row m at offset m(m-1)/2
    s["enc.final_ln.g"] = (d,); s["enc.final_ln.b"] = (d,)
    for m in range(cfg.dec_layers):
        p = f"dec.{m}."
        s[p + "self_ln.g"] = (d,); s[p + "self_ln.b"] = (d,)
        s[p + "self_qkv.w"] = (3 * d, d); s[p + "self_qkv.b"] = (3 * d,)
        s[p + "self_out.w"] = (d, d); s[p + "self_out.b"] = (d,)
        if cfg.use_rpr:
            s[p + "rel_k"] = (R, dh); s[p + "rel_v"] = (R, dh)
        s[p + "cross_ln.g"] = (d,); s[p + "cross_ln.b"] = (d,)
        s[p + "cross_q.w"] = (d, d); s[p + "cross_q.b"] = (d,)
        s[p + "cross_kv.w"] = (2 * d, d); s[p + "cross_kv.b"] = (2 * d,)
        s[p + "cross_out.w"] = (d, d); s[p + "cross_out.b"] = (d,)
        s[p + "ffn_ln.g"] = (d,); s[p + "ffn_ln.b"] = (d,)
        s[p + "ffn1.w"] = (F, d); s[p + "ffn1.b"] = (F,)
        s[p + "ffn2.w"] = (d, F); s[p + "ffn2.b"] = (d,)
    s["dec.final_ln.g"] = (d,); s["dec.final_ln.b"] = (d,)
    return s


def _dlcl_w(cfg: ModelConfig, u: np.ndarray) -> np.ndarray:
    """W[m][k] = (1 + 0.5 (2u-1)) / m for rows m = 1..L+1 (reading R6)."""
    L1 = cfg.enc_layers + 1
    out = np.empty(L1 * (L1 + 1) // 2)
    for m in range(1, L1 + 1):
        o = m * (m - 1) // 2
        out[o:o + m] = (1.0 + 0.5 * (2.0 * u[o:o + m] - 1.0)) / m
    return out


def generate_weights(cfg: ModelConfig, seed: int = WEIGHT_SEED, eos_boost: float = 1.0,
                     dtype=np.float16) -> "OrderedDict[str, np.ndarray]":
    """Return canonical-order dict of FP16-representable tensors (as ``dtype``)."""
    out: "OrderedDict[str, np.ndarray]" = OrderedDict()
    for tid, (name, shape) in enumerate(canonical_shapes(cfg).items()):
        n = int(np.prod(shape))
        u = uniform01(seed, tid, n)
        sym = (2.0 * u - 1.0) * math.sqrt(3.0)  # unit-variance symmetric uniform
        leaf = name.rsplit(".", 1)[-1]
        if name == "emb":
            v = sym / math.sqrt(cfg.d_model)
        elif name == "enc.dlcl.w":
            v = _dlcl_w(cfg, u)
        elif leaf in ("rel_k", "rel_v"):
            v = sym * 0.5
        elif name.endswith("ln.g") or ".ln." in name and leaf == "g":
            v = 1.0 + 0.1 * (2.0 * u - 1.0)
        elif name.endswith("ln.b") or ".ln." in name and leaf == "b":
            v = 0.1 * (2.0 * u - 1.0)
        elif leaf == "w":
            fan_in = shape[1]
            gain = G_DEC if (name.startswith("dec.") and
                             any(t in name for t in (".self_out.", ".cross_out.", ".ffn2."))) else 1.0
            v = sym * gain / math.sqrt(fan_in)
        elif leaf == "b":
            v = sym * 0.02
        else:  # pragma: no cover
            raise KeyError(name)
        v = v.reshape(shape)
        if name == "emb" and eos_boost != 1.0:
            v = v.copy()
            v[EOS_ID] *= eos_boost
        # round once to FP16 so every consumer sees identical values
        out[name] = v.astype(np.float16).astype(dtype)
    return out


def param_count(cfg: ModelConfig, include_dlcl: bool = True) -> int:
    n = 0
    for name, shape in canonical_shapes(cfg).items():
        if not include_dlcl and name.startswith("enc.dlcl."):
            continue
        n += int(np.prod(shape))
    return n
