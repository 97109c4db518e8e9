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
