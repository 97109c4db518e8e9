"""Pins for oracle/model.py + oracle/search.py.

* library pins: with zero RPR tables (and DLCL off) the encoder / decoder equal
  torch.nn.TransformerEncoderLayer / TransformerDecoderLayer(norm_first=True),
  i.e. the pre-norm Transformer of PAPER.md:23 as a textbook library routine.
* reductions: DLCL one-hot with the Eq.2 LN switched off == plain stack
  (reading A22 (i)); W = 0 -> enc == final-LN bias (closed form).
* implementation cross-checks: O-def (loops, no cache) == O-fast (vectorised,
  padded, cached), which pins caching, batching / padding
   and pruning as exact optimisations.
* beam: K >= V^T == exhaustive enumeration; K = 1 == greedy; early stop sound
  (PAPER.md:103).
"""
import math

import numpy as np
import pytest
import torch

from synth import PRESETS, generate_weights, tiny_workload, BOS_ID, EOS_ID
from oracle import OracleModel, greedy_def, translate_fast, beam_search, exhaustive_best
from oracle.nn import sinusoid_pe, log_softmax

TINY = PRESETS["tiny"]


def _zero_rpr(W):
    W = dict(W)
    for k in W:
        if k.endswith("rel_k") or k.endswith("rel_v"):
            W[k] = np.zeros_like(W[k])
    return W


def _t(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float64))


def _set_ln(ln, W, name):
    ln.weight.data = _t(W[name + ".g"]); ln.bias.data = _t(W[name + ".b"])


def test_encoder_equals_torch_prenorm_stack():
    cfg = TINY.replace(use_dlcl=False)
    W = _zero_rpr({k: v.astype(np.float64) for k, v in generate_weights(cfg).items()})
    m = OracleModel(W, cfg)
    src = [17, 400, 5, 999, 23, 3]
    d = cfg.d_model
    x = _t(W["emb"][src] * math.sqrt(d) + sinusoid_pe(len(src), d)).unsqueeze(0)
    for l in range(cfg.enc_layers):
        p = f"enc.{l}."
        lay = torch.nn.TransformerEncoderLayer(d, cfg.n_heads, cfg.d_ffn, dropout=0.0, batch_first=True,
                                               norm_first=True, layer_norm_eps=cfg.ln_eps).double().eval()
        lay.self_attn.in_proj_weight.data = _t(W[p + "qkv.w"]); lay.self_attn.in_proj_bias.data = _t(W[p + "qkv.b"])
        lay.self_attn.out_proj.weight.data = _t(W[p + "out.w"]); lay.self_attn.out_proj.bias.data = _t(W[p + "out.b"])
        lay.linear1.weight.data = _t(W[p + "ffn1.w"]); lay.linear1.bias.data = _t(W[p + "ffn1.b"])
        lay.linear2.weight.data = _t(W[p + "ffn2.w"]); lay.linear2.bias.data = _t(W[p + "ffn2.b"])
        _set_ln(lay.norm1, W, p + "attn_ln"); _set_ln(lay.norm2, W, p + "ffn_ln")
        with torch.no_grad():
            x = lay(x)
    ref = torch.nn.functional.layer_norm(x[0], (d,), _t(W["enc.final_ln.g"]), _t(W["enc.final_ln.b"]), cfg.ln_eps)
    np.testing.assert_allclose(m.encode_def(src), ref.numpy(), rtol=1e-10, atol=1e-10)


def test_decoder_equals_torch_prenorm_layer():
    cfg = TINY.replace(use_dlcl=False)
    W = _zero_rpr({k: v.astype(np.float64) for k, v in generate_weights(cfg).items()})
    m = OracleModel(W, cfg)
    src = [17, 400, 5, 999, 3]
    enc = m.encode_def(src)
    prefix = [BOS_ID, 44, 800, 7, 7, 512]
    d = cfg.d_model
    p = "dec.0."
    lay = torch.nn.TransformerDecoderLayer(d, cfg.n_heads, cfg.d_ffn, dropout=0.0, batch_first=True,
                                           norm_first=True, layer_norm_eps=cfg.ln_eps).double().eval()
    lay.self_attn.in_proj_weight.data = _t(W[p + "self_qkv.w"]); lay.self_attn.in_proj_bias.data = _t(W[p + "self_qkv.b"])
    lay.self_attn.out_proj.weight.data = _t(W[p + "self_out.w"]); lay.self_attn.out_proj.bias.data = _t(W[p + "self_out.b"])
    lay.multihead_attn.in_proj_weight.data = _t(np.concatenate([W[p + "cross_q.w"], W[p + "cross_kv.w"]]))
    lay.multihead_attn.in_proj_bias.data = _t(np.concatenate([W[p + "cross_q.b"], W[p + "cross_kv.b"]]))
    lay.multihead_attn.out_proj.weight.data = _t(W[p + "cross_out.w"]); lay.multihead_attn.out_proj.bias.data = _t(W[p + "cross_out.b"])
    lay.linear1.weight.data = _t(W[p + "ffn1.w"]); lay.linear1.bias.data = _t(W[p + "ffn1.b"])
    lay.linear2.weight.data = _t(W[p + "ffn2.w"]); lay.linear2.bias.data = _t(W[p + "ffn2.b"])
    _set_ln(lay.norm1, W, p + "self_ln"); _set_ln(lay.norm2, W, p + "cross_ln"); _set_ln(lay.norm3, W, p + "ffn_ln")
    T = len(prefix)
    g = _t(W["emb"][prefix] * math.sqrt(d) + sinusoid_pe(T, d)).unsqueeze(0)
    causal = torch.nn.Transformer.generate_square_subsequent_mask(T, dtype=torch.float64)
    with torch.no_grad():
        y = lay(g, _t(enc).unsqueeze(0), tgt_mask=causal)
    h = torch.nn.functional.layer_norm(y[0], (d,), _t(W["dec.final_ln.g"]), _t(W["dec.final_ln.b"]), cfg.ln_eps)
    ref = (h @ _t(W["emb"]).T).numpy()
    for t in range(T):
        np.testing.assert_allclose(m.decoder_logits_def(enc, prefix[:t + 1]), ref[t], rtol=1e-10, atol=1e-10)


def test_dlcl_one_hot_without_ln_is_plain_stack():
    cfg_d = TINY.replace(dlcl_ln=False)
    W = generate_weights(cfg_d)
    L1 = cfg_d.enc_layers + 1
    w = np.zeros(L1 * (L1 + 1) // 2)
    for m_ in range(1, L1 + 1):
        w[m_ * (m_ - 1) // 2 + (m_ - 1)] = 1.0      # W^{(l+1)} = e_l: x_{l+1} = y_l
    W = dict(W); W["enc.dlcl.w"] = w
    plain = {k: v for k, v in W.items() if not k.startswith("enc.dlcl")}
    src = [9, 88, 777, 3]
    a = OracleModel(W, cfg_d).encode_def(src)
    b = OracleModel(plain, TINY.replace(use_dlcl=False)).encode_def(src)
    np.testing.assert_array_equal(a, b)


def test_dlcl_zero_weights_give_final_ln_bias():
    W = dict(generate_weights(TINY))
    W["enc.dlcl.w"] = np.zeros_like(W["enc.dlcl.w"])
    enc = OracleModel(W, TINY).encode_def([5, 6, 7, 3])
    np.testing.assert_allclose(enc, np.tile(W["enc.final_ln.b"].astype(np.float64), (4, 1)), atol=1e-12)


@pytest.fixture(scope="module")
def tiny():
    return OracleModel(generate_weights(TINY, eos_boost=3.0), TINY)


def test_encoder_def_equals_batched(tiny):
    wl = tiny_workload()
    srcs = [wl.sentence(i) for i in range(wl.n)]
    enc, lens = tiny.encode_batch(srcs)
    for i, s in enumerate(srcs):
        np.testing.assert_allclose(enc[i, :len(s)], tiny.encode_def(s), rtol=1e-12, atol=1e-12)


def test_cached_decoder_equals_recompute(tiny):
    wl = tiny_workload()
    srcs = [wl.sentence(i) for i in range(3)]
    enc, lens = tiny.encode_batch(srcs)
    ckv = tiny.cross_kv(enc)
    r = np.random.default_rng(5)
    T = 12  # spans the RPR clip boundary (8/9)
    toks = np.concatenate([np.full((3, 1), BOS_ID), r.integers(4, 1000, size=(3, T - 1))], 1)
    cache = tiny.new_cache(3, T)
    for t in range(T):
        got = tiny.decoder_step(toks[:, t], t, cache, ckv, lens)
        for b in range(3):
            ref = tiny.decoder_logits_def(enc[b, :lens[b]], list(toks[b, :t + 1]))
            np.testing.assert_allclose(got[b], ref, rtol=1e-11, atol=1e-11)


def test_greedy_def_equals_fast_and_prune_invariance(tiny):
    wl = tiny_workload(n=10, seed=3)
    ref = [greedy_def(tiny, wl.sentence(i), wl.caps[i]) for i in range(wl.n)]
    assert any(len(o) < c for o, c in zip(ref, wl.caps)), "eos_boost should produce natural EOS"
    for rho in (0.0, 0.25, 1.0, None):
        for (mt, ms) in ((4096, 512), (40, 3), (16, 1)):
            log = {}
            out = translate_fast(tiny, wl, mt, ms, prune_every=1, prune_ratio=rho, log=log)
            assert out == ref, (rho, mt, ms)
            for bi, t, keep in log["prunes"]:
                assert (np.diff(keep) > 0).all()
    # prune maps exist for rho = 0 on this workload
    log = {}
    translate_fast(tiny, wl, 4096, 512, prune_ratio=0.0, log=log)
    assert len(log["prunes"]) > 0


def test_gen_token_accounting(tiny):
    wl = tiny_workload(n=6, seed=4)
    log = {}
    out = translate_fast(tiny, wl, log=log)
    # generated tokens = output tokens + 1 terminating EOS where one was produced
    n_eos = sum(1 for o, c in zip(out, wl.caps) if len(o) < min(c, 200))
    assert log["gen_tokens"] == sum(len(o) for o in out) + n_eos


# ------------------------------------------------------------------ beam
V8 = TINY.replace(vocab_size=8)


@pytest.fixture(scope="module")
def toy8():
    return OracleModel(generate_weights(V8, seed=77), V8)


@pytest.mark.parametrize("src", [[5, 6, 3], [7, 4, 4, 5, 3]])
def test_beam_full_width_equals_exhaustive(toy8, src):
    cap = 4
    toks_b, sc_b = beam_search(toy8, src, cap, K=8 ** cap)
    toks_e, sc_e = exhaustive_best(toy8, src, cap)
    assert toks_b == toks_e
    assert abs(sc_b - sc_e) < 1e-12


def test_beam_k1_is_greedy(tiny):
    wl = tiny_workload(n=4, seed=9)
    for i in range(wl.n):
        s = wl.sentence(i)
        assert beam_search(tiny, s, wl.caps[i], K=1)[0] == greedy_def(tiny, s, wl.caps[i])


@pytest.mark.parametrize("K", [2, 3, 4])
def test_beam_early_stop_is_sound(toy8, K):
    r = np.random.default_rng(K)
    for _ in range(4):
        src = list(r.integers(4, 8, size=r.integers(1, 6))) + [EOS_ID]
        a = beam_search(toy8, src, 6, K=K, early_stop=True)
        b = beam_search(toy8, src, 6, K=K, early_stop=False)
        assert a[0] == b[0] and abs(a[1] - b[1]) < 1e-12


def _torch_layer(W, cfg, l):
    """torch.nn.TransformerEncoderLayer(norm_first) loaded with encoder layer l (zero RPR)."""
    d = cfg.d_model
    p = f"enc.{l}."
    lay = torch.nn.TransformerEncoderLayer(d, cfg.n_heads, cfg.d_ffn, dropout=0.0, batch_first=True,
                                           norm_first=True, layer_norm_eps=cfg.ln_eps).double().eval()
    lay.self_attn.in_proj_weight.data = _t(W[p + "qkv.w"]); lay.self_attn.in_proj_bias.data = _t(W[p + "qkv.b"])
    lay.self_attn.out_proj.weight.data = _t(W[p + "out.w"]); lay.self_attn.out_proj.bias.data = _t(W[p + "out.b"])
    lay.linear1.weight.data = _t(W[p + "ffn1.w"]); lay.linear1.bias.data = _t(W[p + "ffn1.b"])
    lay.linear2.weight.data = _t(W[p + "ffn2.w"]); lay.linear2.bias.data = _t(W[p + "ffn2.b"])
    _set_ln(lay.norm1, W, p + "attn_ln"); _set_ln(lay.norm2, W, p + "ffn_ln")
    return lay


# DLCL weight rows W^{(m)}, m = 1..L+1 (L = 2), written out by hand
_DLCL_CASES = {
    # W^{(l+1)} = 1/(l+1) . 1  ->  x_{l+1} = mean of z_0..z_l (SURVEY §8(c) DLCL pins)
    "uniform_mean": [[1.0], [0.5, 0.5], [1 / 3, 1 / 3, 1 / 3]],
    # the [.5, .25, .25] hand sum for the encoder top: x_3 = .5 z_0 + .25 z_1 + .25 z_2
    "hand_sum": [[0.75], [0.3, 0.7], [0.5, 0.25, 0.25]],
    # reading A22 (ii): one-hot W^{(l+1)} = e_l with the Eq.-2 LN ON == the plain pre-norm
    # stack with an explicit LN^dl_l inserted after every layer (and before the final LN)
    "one_hot_ln_on": [[1.0], [0.0, 1.0], [0.0, 0.0, 1.0]],
}


@pytest.mark.parametrize("case", sorted(_DLCL_CASES))
def test_dlcl_eq2_against_torch_layers(case):
    """Eq. 1-2: z_k = LN^dl_k(y_k), x_{l+1} = sum_{k<=l} W^{(l+1)}_k z_k,
    enc = LN^enc(sum_k W^{(L+1)}_k z_k), evaluated here step by step with torch layers and
    F.layer_norm on hand-written weight rows (zero RPR tables so the layers are the textbook
    pre-norm TransformerEncoderLayer)."""
    cfg = TINY  # L = 2, DLCL on, dlcl_ln on
    rows = _DLCL_CASES[case]
    W = _zero_rpr({k: v.astype(np.float64) for k, v in generate_weights(cfg).items()})
    W["enc.dlcl.w"] = np.concatenate([np.array(r, dtype=np.float64) for r in rows])
    src = [17, 400, 5, 999, 23, 3]
    d = cfg.d_model
    ln = lambda x, name: torch.nn.functional.layer_norm(x, (d,), _t(W[name + ".g"]), _t(W[name + ".b"]),
                                                        cfg.ln_eps)
    y = _t(W["emb"][src] * math.sqrt(d) + sinusoid_pe(len(src), d)).unsqueeze(0)
    zs = [ln(y, "enc.dlcl.ln.0")]
    x = rows[0][0] * zs[0]
    with torch.no_grad():
        for l in range(cfg.enc_layers):
            y = _torch_layer(W, cfg, l)(x)
            zs.append(ln(y, f"enc.dlcl.ln.{l + 1}"))
            x = sum(wk * zk for wk, zk in zip(rows[l + 1], zs))
    ref = ln(x[0], "enc.final_ln").numpy()
    got = OracleModel(W, cfg).encode_def(src)
    np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-10)
    if case == "uniform_mean":   # the combination really is the mean of the z_k
        np.testing.assert_allclose(x.numpy(), (sum(zs) / 3).numpy(), rtol=1e-14, atol=1e-14)
    if case == "one_hot_ln_on":
        # == plain stack with LN^dl between layers (no DLCL weights anywhere)
        with torch.no_grad():
            h = ln(_t(W["emb"][src] * math.sqrt(d) + sinusoid_pe(len(src), d)).unsqueeze(0), "enc.dlcl.ln.0")
            for l in range(cfg.enc_layers):
                h = ln(_torch_layer(W, cfg, l)(h), f"enc.dlcl.ln.{l + 1}")
        np.testing.assert_allclose(got, ln(h[0], "enc.final_ln").numpy(), rtol=1e-10, atol=1e-10)
