"""ORACLE (test infrastructure only) — elementary operators, FP64 by default.

Each function restates one definition:
  * layer_norm — Ba et al., used pre-norm ("proper use of layer
    normalization"); population variance, eps = 1e-5 (reading R10).
    Pinned by tests/test_oracle_nn.py (closed forms; torch.nn.functional.layer_norm).
  * softmax / log_softmax — FP32-or-wider normaliser ("all operations related
    to reduce_sum" in high precision). Pinned: closed forms.
  * sinusoid_pe — absolute positions, "maximum position ... 1024",
    fairseq layout (reading R8). Pinned: PE(0), PE(p)[0] = sin p, PE(p)[d/2] = cos p.
  * rel_index — Shaw et al. clipped distance, "maximum relative length was 8"
    (reading R7/R24). Pinned: brute-force table.
  * rpr_attention_loops — Shaw et al. relative self-attention written as the
    plain double loop over (query i, key j); keys AND values get the clipped
    relative embedding (reading R7). Pinned (tests/test_oracle_nn.py): zero tables ==
    torch scaled_dot_product_attention (test_rpr_zero_tables_is_vanilla_attention);
    constant tables == vanilla + shift (test_rpr_constant_tables_shift); n = 1 closed
    form o = v_0 + A^V[k] (test_rpr_single_token_closed_form); the j - i DIRECTION by a
    hand-computed asymmetric-table example, n = 3, k = 1 (test_rpr_direction_hand_example);
    the unclipped case k >= n - 1 with distance-linear tables == SDPA on position-shifted
    keys / values (test_rpr_unclipped_linear_tables_are_shifted_vanilla).
"""
from __future__ import annotations

import math

import numpy as np


def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def softmax(x: np.ndarray, axis: int = -1) -> np.ndarray:
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=axis, keepdims=True)


def log_softmax(x: np.ndarray, axis: int = -1) -> np.ndarray:
    m = np.max(x, axis=axis, keepdims=True)
    return x - m - np.log(np.exp(x - m).sum(axis=axis, keepdims=True))


def sinusoid_pe(n_pos: int, d: int, dtype=np.float64) -> np.ndarray:
    """PE(p)[i] = sin(p w_i), PE(p)[d/2+i] = cos(p w_i), w_i = exp(-ln(1e4) i/(d/2-1))."""
    half = d // 2
    w = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float64) / (half - 1))
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * w[None, :]
    return np.concatenate([np.sin(ang), np.cos(ang)], axis=1).astype(dtype)


def rel_index(i: int, j: int, k: int) -> int:
    """r(i, j) = clip(j - i, -k, k) + k  in [0, 2k]."""
    return min(max(j - i, -k), k) + k


def rpr_attention_loops(q, kk, v, ak, av, n_heads: int, kclip: int, allowed) -> np.ndarray:
    """Relative-position multi-head attention, plain loops.

    q: [nq, d] queries at positions qpos (given implicitly by ``allowed``);
    kk, v: [nk, d]; ak, av: [2k+1, dh] or None (no RPR).
    ``allowed(i, j) -> (bool, query_position)`` decides masking.
      e_ij = q_i . (k_j + A^K[r(i,j)]) / sqrt(dh)
      o_i  = sum_j softmax_j(e_i)_j (v_j + A^V[r(i,j)])
    """
    nq, d = q.shape
    dh = d // n_heads
    out = np.zeros((nq, d), dtype=q.dtype)
    scale = 1.0 / math.sqrt(dh)
    for h in range(n_heads):
        sl = slice(h * dh, (h + 1) * dh)
        for i in range(nq):
            js, rs, es = [], [], []
            for j in range(kk.shape[0]):
                ok, qpos = allowed(i, j)
                if not ok:
                    continue
                r = rel_index(qpos, j, kclip)
                key = kk[j, sl].astype(np.float64)
                if ak is not None:
                    key = key + ak[r]
                js.append(j)
                rs.append(r)
                es.append(float(np.dot(q[i, sl], key)) * scale)
            es = np.array(es, dtype=np.float64)
            a = np.exp(es - es.max())
            a = a / a.sum()
            acc = np.zeros(dh, dtype=np.float64)
            for aj, j, r in zip(a, js, rs):
                val = v[j, sl].astype(np.float64)
                if av is not None:
                    val = val + av[r]
                acc += aj * val
            out[i, sl] = acc
    return out
