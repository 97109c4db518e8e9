"""ORACLE (test infrastructure only) — the Transformer-DLCL-RPR of PAPER.md.

Two implementations of the same model, so each pins the other:

* **O-def** (``encode_def``, ``decoder_logits_def``): one sentence, plain
  loops for attention (``oracle.nn.rpr_attention_loops``), explicit DLCL sum,
  decoder step t recomputes the whole prefix 0..t (no cache).
* **O-fast** (``encode_batch``, ``decoder_step``): padded batches, vectorised
  attention, cached decoder self-attention K/V and cross K/V projected once
  per sentence ("we cache the linear transformations for keys and values
  before the self-attention and cross-attention layers").

Model (readings R1-R11):
  * embedding  y0[p] = sqrt(d) E[s_p] + PE(p)      tied E
  * encoder layer l (pre-norm):
        a   = x_l + W_o RPRAttn(LN^a_l(x_l)) + b_o
        y_l = a + FFN_l(LN^f_l(a)),  FFN(u) = max(0, u W1^T + b1) W2^T + b2
  * DLCL (Eq. 1-2):
        z_k = LN^dl_k(y_k);  x_{l+1} = sum_{k=0..l} W^{(l+1)}_k z_k
        enc = LN^enc(sum_{k=0..L} W^{(L+1)}_k z_k)              (reading R4)
    without DLCL: x_1 = y_0, x_{l+1} = y_l, enc = LN^enc(y_L).
  * decoder step t (w_0 = BOS):  g = sqrt(d) E[w_t] + PE(t); per layer
        g += SelfAttn_RPR(LN^s(g)) over positions 0..t (causal)
        g += W_co CrossAttn(LN^c(g) W_q^T + b, CK, CV) + b_co   (no RPR, R7)
        g += FFN(LN^f(g))
    h = LN^dec(g), logits = h E^T (tied, no bias).

Parity pins (tests/test_oracle_model.py): encoder layer == torch
TransformerEncoderLayer(norm_first) with zero RPR tables
(test_encoder_equals_torch_prenorm_stack); decoder layer == torch
TransformerDecoderLayer(norm_first) with zero tables
(test_decoder_equals_torch_prenorm_layer); O-def == O-fast
(test_encoder_def_equals_batched, test_cached_decoder_equals_recompute,
test_greedy_def_equals_fast_and_prune_invariance); DLCL (encode_def's Eq. 2 sum,
test_dlcl_eq2_against_torch_layers): uniform W -> mean of z_k, the [.5,.25,.25]
hand sum, one-hot W with LN^dl on == plain stack + explicit LN^dl (A22 ii);
one-hot with LN^dl off == plain stack (A22 i,
test_dlcl_one_hot_without_ln_is_plain_stack); W = 0 -> final-LN bias;
parameter counts == PAPER.md Tables 1-2 (tests/test_oracle_params.py).
"""
from __future__ import annotations

import math

import numpy as np

from .nn import layer_norm, softmax, sinusoid_pe, rpr_attention_loops


class OracleModel:
    def __init__(self, weights: dict, cfg, dtype=np.float64):
        self.cfg = cfg
        self.dt = dtype
        self.W = {k: np.asarray(v, dtype=dtype) for k, v in weights.items()}
        self.pe = sinusoid_pe(cfg.max_pos, cfg.d_model, dtype)
        self.emb_scale = dtype(math.sqrt(cfg.d_model))
        L1 = cfg.enc_layers + 1
        if cfg.use_dlcl:
            wflat = self.W["enc.dlcl.w"]
            # row m (1..L+1) holds W^{(m)}_k, k = 0..m-1, at offset m(m-1)/2
            self.dlcl = [None] + [wflat[m * (m - 1) // 2: m * (m - 1) // 2 + m] for m in range(1, L1 + 1)]

    # ------------------------------------------------------------------ helpers
    def _ln(self, x, name):
        return layer_norm(x, self.W[name + ".g"], self.W[name + ".b"], self.cfg.ln_eps)

    def _lin(self, x, name):
        return x @ self.W[name + ".w"].T + self.W[name + ".b"]

    def _ffn(self, u, p):
        return self._lin(np.maximum(self._lin(u, p + "ffn1"), 0.0), p + "ffn2")

    def _rel(self, p):
        if not self.cfg.use_rpr:
            return None, None
        return self.W[p + "rel_k"], self.W[p + "rel_v"]

    def embed(self, ids, positions):
        return self.W["emb"][np.asarray(ids)] * self.emb_scale + self.pe[np.asarray(positions)]

    def _dlcl_z(self, y, k):
        return self._ln(y, f"enc.dlcl.ln.{k}") if self.cfg.dlcl_ln else y

    # ------------------------------------------------------------ O-def encoder
    def encode_def(self, src) -> np.ndarray:
        """One sentence -> enc [n, d]; plain-loop attention, explicit DLCL."""
        cfg = self.cfg
        n = len(src)
        y0 = self.embed(src, np.arange(n))
        zs = []
        if cfg.use_dlcl:
            zs.append(self._dlcl_z(y0, 0))
            x = self.dlcl[1][0] * zs[0]
        else:
            x = y0
        for l in range(cfg.enc_layers):
            p = f"enc.{l}."
            u = self._ln(x, p + "attn_ln")
            qkv = self._lin(u, p + "qkv")
            d = cfg.d_model
            ak, av = self._rel(p)
            o = rpr_attention_loops(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], ak, av,
                                    cfg.n_heads, cfg.max_rel_pos, lambda i, j: (True, i))
            a = x + self._lin(o, p + "out")
            y = a + self._ffn(self._ln(a, p + "ffn_ln"), p)
            if cfg.use_dlcl:
                zs.append(self._dlcl_z(y, l + 1))
                w = self.dlcl[l + 2]
                x = np.zeros_like(y)
                for k in range(l + 2):          # Eq. 2: sum_{k=0..l} (1-based l+1)
                    x = x + w[k] * zs[k]
            else:
                x = y
        return self._ln(x, "enc.final_ln")

    # ------------------------------------------------------------ O-def decoder
    def decoder_logits_def(self, enc: np.ndarray, prefix) -> np.ndarray:
        """Logits at the last position of ``prefix`` (w_0 = BOS, ..., w_t), recomputing
        every position 0..t from scratch (no cache)."""
        cfg = self.cfg
        d = cfg.d_model
        T = len(prefix)
        g = self.embed(prefix, np.arange(T))
        for m in range(cfg.dec_layers):
            p = f"dec.{m}."
            u = self._ln(g, p + "self_ln")
            qkv = self._lin(u, p + "self_qkv")
            ak, av = self._rel(p)
            o = rpr_attention_loops(qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:], ak, av,
                                    cfg.n_heads, cfg.max_rel_pos, lambda i, j: (j <= i, i))
            g = g + self._lin(o, p + "self_out")
            u = self._ln(g, p + "cross_ln")
            q = self._lin(u, p + "cross_q")
            kv = self._lin(enc, p + "cross_kv")
            o = rpr_attention_loops(q, kv[:, :d], kv[:, d:], None, None, cfg.n_heads,
                                    cfg.max_rel_pos, lambda i, j: (True, i))
            g = g + self._lin(o, p + "cross_out")
            g = g + self._ffn(self._ln(g, p + "ffn_ln"), p)
        h = self._ln(g[-1], "dec.final_ln")
        return h @ self.W["emb"].T

    # ----------------------------------------------------------- O-fast encoder
    def _mha_vec(self, q, k, v, ak, av, key_mask, qpos, kpos):
        """Vectorised RPR attention. q [B,Sq,d], k/v [B,Sk,d], key_mask [B,Sk] bool
        (True = attend), qpos [Sq] / kpos [Sk] absolute positions for r(i,j)."""
        cfg = self.cfg
        B, Sq, d = q.shape
        Sk = k.shape[1]
        H, dh = cfg.n_heads, cfg.d_head
        qh = q.reshape(B, Sq, H, dh).transpose(0, 2, 1, 3)
        kh = k.reshape(B, Sk, H, dh).transpose(0, 2, 1, 3)
        vh = v.reshape(B, Sk, H, dh).transpose(0, 2, 1, 3)
        e = qh @ kh.transpose(0, 1, 3, 2)                      # [B,H,Sq,Sk]
        if ak is not None:
            kc = cfg.max_rel_pos
            R = np.clip(kpos[None, :] - qpos[:, None], -kc, kc) + kc  # [Sq,Sk]
            qa = qh @ ak.T                                      # [B,H,Sq,2k+1]
            e = e + np.take_along_axis(qa, np.broadcast_to(R, (B, H, Sq, Sk)), axis=3)
        e = e / math.sqrt(dh)
        mask = np.broadcast_to(key_mask[:, None, None, :], e.shape)
        e = np.where(mask, e, -np.inf)
        a = softmax(e, axis=-1)
        o = a @ vh                                              # [B,H,Sq,dh]
        if av is not None:
            onehot = np.eye(2 * kc + 1, dtype=self.dt)[R]       # [Sq,Sk,2k+1]
            bucket = np.einsum("bhij,ijr->bhir", a, onehot)
            o = o + bucket @ av
        return o.transpose(0, 2, 1, 3).reshape(B, Sq, d)

    def encode_batch(self, srcs):
        """Padded batch -> (enc [B,S,d], src_len [B]); padding rows are PAD ids."""
        cfg = self.cfg
        B = len(srcs)
        lens = np.array([len(s) for s in srcs])
        S = int(lens.max())
        ids = np.zeros((B, S), dtype=np.int64)
        for b, s in enumerate(srcs):
            ids[b, :len(s)] = s
        kmask = np.arange(S)[None, :] < lens[:, None]
        pos = np.arange(S)
        y0 = self.embed(ids, pos[None, :].repeat(B, 0))
        d = cfg.d_model
        zs = []
        if cfg.use_dlcl:
            zs.append(self._dlcl_z(y0, 0))
            x = self.dlcl[1][0] * zs[0]
        else:
            x = y0
        for l in range(cfg.enc_layers):
            p = f"enc.{l}."
            qkv = self._lin(self._ln(x, p + "attn_ln"), p + "qkv")
            ak, av = self._rel(p)
            o = self._mha_vec(qkv[..., :d], qkv[..., d:2 * d], qkv[..., 2 * d:], ak, av, kmask, pos, pos)
            a = x + self._lin(o, p + "out")
            y = a + self._ffn(self._ln(a, p + "ffn_ln"), p)
            if cfg.use_dlcl:
                zs.append(self._dlcl_z(y, l + 1))
                w = self.dlcl[l + 2]
                x = sum(w[k] * zs[k] for k in range(l + 2))
            else:
                x = y
        return self._ln(x, "enc.final_ln"), lens

    def cross_kv(self, enc):
        """Cross K/V for every decoder layer, once per sentence."""
        d = self.cfg.d_model
        out = []
        for m in range(self.cfg.dec_layers):
            kv = self._lin(enc, f"dec.{m}.cross_kv")
            out.append((kv[..., :d], kv[..., d:]))
        return out

    # ----------------------------------------------------------- O-fast decoder
    def new_cache(self, B, T):
        cfg = self.cfg
        return [(np.zeros((B, T, cfg.d_model), self.dt), np.zeros((B, T, cfg.d_model), self.dt))
                for _ in range(cfg.dec_layers)]

    def decoder_step(self, tokens, t, self_cache, ckv, src_len):
        """Cached step t for rows of one batch: tokens [B] (w_t), caches indexed by row.
        Appends k_t, v_t to ``self_cache`` and returns logits [B, V]."""
        cfg = self.cfg
        d = cfg.d_model
        B = len(tokens)
        g = self.embed(tokens, np.full(B, t))[:, None, :]       # [B,1,d]
        pos_q = np.array([t])
        for m in range(cfg.dec_layers):
            p = f"dec.{m}."
            qkv = self._lin(self._ln(g, p + "self_ln"), p + "self_qkv")
            Kc, Vc = self_cache[m]
            Kc[:, t] = qkv[:, 0, d:2 * d]
            Vc[:, t] = qkv[:, 0, 2 * d:]
            ak, av = self._rel(p)
            o = self._mha_vec(qkv[..., :d], Kc[:, :t + 1], Vc[:, :t + 1], ak, av,
                              np.ones((B, t + 1), bool), pos_q, np.arange(t + 1))
            g = g + self._lin(o, p + "self_out")
            q = self._lin(self._ln(g, p + "cross_ln"), p + "cross_q")
            CK, CV = ckv[m]
            S = CK.shape[1]
            kmask = np.arange(S)[None, :] < src_len[:, None]
            o = self._mha_vec(q, CK, CV, None, None, kmask, pos_q, np.arange(S))
            g = g + self._lin(o, p + "cross_out")
            g = g + self._ffn(self._ln(g, p + "ffn_ln"), p)
        h = self._ln(g[:, 0], "dec.final_ln")
        return h @ self.W["emb"].T
