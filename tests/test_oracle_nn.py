"""Pins for oracle/nn.py against closed forms, special cases and library routines."""
import math

import numpy as np
import pytest
import torch

from oracle.nn import layer_norm, softmax, log_softmax, sinusoid_pe, rel_index, rpr_attention_loops

EPS = 1e-5


def test_layer_norm_closed_forms():
    # SPEC.md:78-81 examples (eps = 1e-5 reading R10)
    np.testing.assert_allclose(layer_norm(np.array([1., 1, 1]), 1.0, 0.0, EPS), [0, 0, 0], atol=0)
    v = 1.0 / math.sqrt(1.0 + EPS)
    np.testing.assert_allclose(layer_norm(np.array([1., -1]), 1.0, 0.0, EPS), [v, -v], rtol=1e-15)
    np.testing.assert_allclose(layer_norm(np.array([2., 4]), 0.0, 7.0, EPS), [7, 7], atol=0)


def test_layer_norm_vs_torch():
    r = np.random.default_rng(0)
    x = r.normal(size=(5, 64)) * 3 + 1
    g, b = r.normal(size=64), r.normal(size=64)
    ref = torch.nn.functional.layer_norm(torch.from_numpy(x), (64,), torch.from_numpy(g),
                                         torch.from_numpy(b), eps=EPS).numpy()
    np.testing.assert_allclose(layer_norm(x, g, b, EPS), ref, rtol=1e-12, atol=1e-12)


def test_softmax_closed_forms():
    # SPEC.md:69-72
    np.testing.assert_allclose(softmax(np.zeros(4)), [0.25] * 4, rtol=1e-15)
    np.testing.assert_allclose(softmax(np.array([5.0, -np.inf])), [1.0, 0.0], atol=0)
    np.testing.assert_allclose(softmax(np.array([0.0, math.log(2)])), [1 / 3, 2 / 3], rtol=1e-15)


def test_log_softmax_vs_torch_and_argmax():
    r = np.random.default_rng(1)
    x = r.normal(size=(7, 1000)) * 4
    ref = torch.log_softmax(torch.from_numpy(x), -1).numpy()
    np.testing.assert_allclose(log_softmax(x), ref, rtol=1e-12, atol=1e-12)
    # removing log_softmax does not change the greedy choice
    assert (np.argmax(x, 1) == np.argmax(log_softmax(x), 1)).all()
    assert (np.argmax(x + 3.7, 1) == np.argmax(x, 1)).all()
    # ties -> lowest index (reading R13)
    assert int(np.argmax(np.array([5.0, 5.0]))) == 0


def test_sinusoid_special_values():
    d = 512
    pe = sinusoid_pe(1024, d)
    h = d // 2
    np.testing.assert_array_equal(pe[0, :h], 0.0)       # sin 0
    np.testing.assert_array_equal(pe[0, h:], 1.0)       # cos 0
    p = np.arange(1024)
    np.testing.assert_allclose(pe[:, 0], np.sin(p), rtol=0, atol=1e-12)       # w_0 = 1
    np.testing.assert_allclose(pe[:, h], np.cos(p), rtol=0, atol=1e-12)
    np.testing.assert_allclose(pe[:, h - 1], np.sin(p * 1e-4), rtol=1e-9, atol=1e-15)  # w_{h-1}=1e-4
    np.testing.assert_allclose(pe[:, :h] ** 2 + pe[:, h:] ** 2, 1.0, atol=1e-12)


def test_rel_index_table():
    # k = 2: r(i,j) = clip(j-i,-2,2)+2 written out by hand for i,j in 0..4
    exp = np.array([[2, 3, 4, 4, 4],
                    [1, 2, 3, 4, 4],
                    [0, 1, 2, 3, 4],
                    [0, 0, 1, 2, 3],
                    [0, 0, 0, 1, 2]])
    got = np.array([[rel_index(i, j, 2) for j in range(5)] for i in range(5)])
    np.testing.assert_array_equal(got, exp)
    # k = 8 boundary (reading R24): distances +-8 are the last distinct buckets
    assert rel_index(0, 8, 8) == 16 and rel_index(0, 9, 8) == 16 and rel_index(0, 7, 8) == 15
    assert rel_index(9, 0, 8) == 0 and rel_index(8, 0, 8) == 0 and rel_index(7, 0, 8) == 1


def _sdpa(q, k, v, H, mask):
    n, d = q.shape
    dh = d // H
    t = lambda a: torch.from_numpy(a).reshape(a.shape[0], H, dh).transpose(0, 1)
    o = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v), attn_mask=torch.from_numpy(mask))
    return o.transpose(0, 1).reshape(n, d).numpy()


@pytest.mark.parametrize("causal", [False, True])
def test_rpr_zero_tables_is_vanilla_attention(causal):
    r = np.random.default_rng(2)
    n, d, H = 11, 32, 4
    q, k, v = (r.normal(size=(n, d)) for _ in range(3))
    z = np.zeros((17, d // H))
    mask = np.tril(np.ones((n, n), bool)) if causal else np.ones((n, n), bool)
    if not causal:
        mask[:, 9:] = False  # encoder-style key padding mask
    got = rpr_attention_loops(q, k, v, z, z, H, 8, lambda i, j: (bool(mask[i, j]), i))
    np.testing.assert_allclose(got, _sdpa(q, k, v, H, mask), rtol=1e-12, atol=1e-12)


def test_rpr_constant_tables_shift():
    """A^K rows all equal: softmax is shift invariant -> vanilla; A^V rows all c -> vanilla + c."""
    r = np.random.default_rng(3)
    n, d, H = 9, 32, 4
    q, k, v = (r.normal(size=(n, d)) for _ in range(3))
    c = r.normal(size=d // H)
    ak = np.tile(r.normal(size=d // H), (17, 1))
    av = np.tile(c, (17, 1))
    got = rpr_attention_loops(q, k, v, ak, av, H, 8, lambda i, j: (True, i))
    ref = _sdpa(q, k, v, H, np.ones((n, n), bool)) + np.tile(c, H)
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_rpr_single_token_closed_form():
    r = np.random.default_rng(4)
    d, H = 32, 4
    q, k, v = (r.normal(size=(1, d)) for _ in range(3))
    ak, av = r.normal(size=(17, 8)), r.normal(size=(17, 8))
    got = rpr_attention_loops(q, k, v, ak, av, H, 8, lambda i, j: (True, i))
    np.testing.assert_allclose(got[0], v[0] + np.tile(av[8], H), rtol=1e-14)  # o = v_0 + A^V[k]


def test_rpr_direction_hand_example():
    """Shaw et al. (cited at PAPER.md:23): a^K_ij = w^K_clip(j-i, k), e_ij = q_i.(k_j + a^K_ij)/sqrt(dz),
    o_i = sum_j a_ij (v_j + a^V_ij).  Hand example with an ASYMMETRIC table, so a swapped
    clip(i-j) gather fails: n = 3, k = 1, H = 1, dh = 2, q_i = e_0, k_j = v_j = 0,
    A^K[r] = (r - k) e_0  ->  e_ij = clip(j-i, -1, 1)/sqrt(2);
    A^V = [[1, 0], [0, 1], [1, 1]] (bucket of distance -1, 0, +1)."""
    s = 1.0 / math.sqrt(2.0)
    q = np.array([[1.0, 0.0]] * 3)
    z = np.zeros((3, 2))
    ak = np.array([[-1.0, 0.0], [0.0, 0.0], [1.0, 0.0]])
    av = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    got = rpr_attention_loops(q, z, z, ak, av, 1, 1, lambda i, j: (True, i))
    E = math.exp(s)
    Ei = math.exp(-s)
    # i = 0: distances 0, +1, +2 -> buckets 1, 2, 2; logits 0, s, s
    o0 = (1.0 * av[1] + 2 * E * av[2]) / (1.0 + 2 * E)
    # i = 1: distances -1, 0, +1 -> buckets 0, 1, 2; logits -s, 0, s
    o1 = (Ei * av[0] + 1.0 * av[1] + E * av[2]) / (Ei + 1.0 + E)
    # i = 2: distances -2, -1, 0 -> buckets 0, 0, 1; logits -s, -s, 0
    o2 = (2 * Ei * av[0] + 1.0 * av[1]) / (2 * Ei + 1.0)
    np.testing.assert_allclose(got, np.array([o0, o1, o2]), rtol=1e-14, atol=1e-15)
    # the causal (decoder) mask keeps only j <= i: row 2 is unchanged, row 0 = A^V[k]
    got_c = rpr_attention_loops(q, z, z, ak, av, 1, 1, lambda i, j: (j <= i, i))
    np.testing.assert_allclose(got_c[0], av[1], rtol=1e-15)
    np.testing.assert_allclose(got_c[2], o2, rtol=1e-14)


@pytest.mark.parametrize("causal", [False, True])
def test_rpr_unclipped_linear_tables_are_shifted_vanilla(causal):
    """Unclipped case (k >= n-1: every distance j-i has its own bucket j-i+k).  With tables
    linear in the distance, A^K[r] = (r-k) u and A^V[r] = (r-k) w:
      e_ij = q_i.(k_j + j u)/sqrt(dh) - i q_i.u/sqrt(dh)   (the last term is constant in j:
                                                           softmax ignores it)
      o_i  = sum_j a_ij (v_j + j w) - i w.
    So RPR == torch scaled_dot_product_attention on keys k_j + j u, values v_j + j w, minus
    i w — a library routine pin that fixes both the direction j - i and the bucket offset."""
    r = np.random.default_rng(8)
    n, d, H, kc = 9, 32, 4, 8
    dh = d // H
    q, k, v = (r.normal(size=(n, d)) for _ in range(3))
    u, w = r.normal(size=dh) * 0.3, r.normal(size=dh)
    dist = np.arange(2 * kc + 1) - kc
    ak, av = dist[:, None] * u[None, :], dist[:, None] * w[None, :]
    mask = np.tril(np.ones((n, n), bool)) if causal else np.ones((n, n), bool)
    got = rpr_attention_loops(q, k, v, ak, av, H, kc, lambda i, j: (bool(mask[i, j]), i))
    pos = np.arange(n)[:, None]
    ks = k + pos * np.tile(u, H)
    vs = v + pos * np.tile(w, H)
    ref = _sdpa(q, ks, vs, H, mask) - pos * np.tile(w, H)
    np.testing.assert_allclose(got, ref, rtol=1e-11, atol=1e-11)
    # with a clip (k = 2 < n - 1) the same tables are NOT the shifted vanilla attention
    got2 = rpr_attention_loops(q, k, v, ak[kc - 2:kc + 3], av[kc - 2:kc + 3], H, 2,
                               lambda i, j: (bool(mask[i, j]), i))
    assert np.abs(got2 - ref).max() > 1e-3
