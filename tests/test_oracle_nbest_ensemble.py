"""Pins for the §8(f) oracle rows (CPU): N-best beam search (the 4-best lists of
sequence-level KD; reading R27) and the teacher-ensemble step distribution
(reading R26).

* N-best with K >= V^T equals brute-force enumeration of every complete sequence;
* N = 1 is the 1-best beam search; early stop on == off (sound for non-increasing scores);
* the N-best list is score-sorted and its sequences are distinct;
* an ensemble of M copies of one model is that model (log-probs within 1e-12); the
  ensemble distribution is a distribution (sums to 1); the full-width ensemble beam equals
  brute force over the averaged distribution."""
import math

import numpy as np
import pytest

from synth import generate_weights
from synth.config import EOS_ID, PRESETS
from oracle import (OracleModel, beam_search, beam_search_nbest, exhaustive_nbest,
                    ensemble_step_logprobs)

TINY = PRESETS["tiny"]
V8 = TINY.replace(vocab_size=8)


@pytest.fixture(scope="module")
def toy8():
    return OracleModel(generate_weights(V8, seed=77), V8)


@pytest.fixture(scope="module")
def toy8b():
    return OracleModel(generate_weights(V8, seed=78), V8)


@pytest.mark.parametrize("src,N", [([5, 6, 3], 4), ([7, 4, 4, 5, 3], 3), ([6, 3], 2)])
def test_nbest_full_width_equals_exhaustive(toy8, src, N):
    cap = 4
    got = beam_search_nbest(toy8, src, cap, K=8 ** cap, nbest=N)
    ref = exhaustive_nbest(toy8, src, cap, N)
    assert [t for t, _ in got] == [t for t, _ in ref]
    assert all(abs(a[1] - b[1]) < 1e-12 for a, b in zip(got, ref))


@pytest.mark.parametrize("K,N", [(2, 2), (4, 4), (4, 2), (3, 1)])
def test_nbest_early_stop_is_sound(toy8, K, N):
    r = np.random.default_rng(10 * K + N)
    for _ in range(4):
        src = list(r.integers(4, 8, size=r.integers(1, 6))) + [EOS_ID]
        a = beam_search_nbest(toy8, src, 6, K=K, nbest=N, early_stop=True)
        b = beam_search_nbest(toy8, src, 6, K=K, nbest=N, early_stop=False)
        assert [t for t, _ in a] == [t for t, _ in b]
        assert all(abs(x[1] - y[1]) < 1e-12 for x, y in zip(a, b))


def test_nbest_one_is_beam(toy8):
    for src in ([5, 6, 3], [4, 4, 7, 3]):
        assert beam_search_nbest(toy8, src, 5, K=3, nbest=1)[0] == beam_search(toy8, src, 5, K=3)


def test_nbest_sorted_and_distinct(toy8):
    got = beam_search_nbest(toy8, [5, 5, 6, 7, 3], 6, K=4, nbest=4)
    sc = [s for _, s in got]
    assert sc == sorted(sc, reverse=True)
    assert len({tuple(t) for t, _ in got}) == len(got)


def test_ensemble_of_copies_is_the_model(toy8):
    src = [5, 6, 7, 3]
    one = ensemble_step_logprobs([toy8], src)
    three = ensemble_step_logprobs([toy8, toy8, toy8], src)
    prefixes = [[2], [2, 5], [2, 5, 6]]
    assert np.abs(one(prefixes) - three(prefixes)).max() < 1e-12
    a = beam_search(toy8, src, 5, K=4)
    b = beam_search(toy8, src, 5, K=4, step_logprobs=three)
    assert a[0] == b[0] and abs(a[1] - b[1]) < 1e-12


def test_ensemble_is_an_average_of_distributions(toy8, toy8b):
    src = [4, 7, 3]
    ens = ensemble_step_logprobs([toy8, toy8b], src)
    m1 = ensemble_step_logprobs([toy8], src)
    m2 = ensemble_step_logprobs([toy8b], src)
    pre = [[2, 4], [2]]
    e = np.exp(ens(pre))
    assert np.abs(e.sum(axis=1) - 1.0).max() < 1e-12
    assert np.abs(e - 0.5 * (np.exp(m1(pre)) + np.exp(m2(pre)))).max() < 1e-12


def test_ensemble_full_width_beam_equals_exhaustive(toy8, toy8b):
    src = [6, 5, 3]
    cap = 3
    ens = ensemble_step_logprobs([toy8, toy8b], src)
    got = beam_search_nbest(toy8, src, cap, K=8 ** cap, nbest=2, step_logprobs=ens)
    ref = exhaustive_nbest(toy8, src, cap, 2, step_logprobs=ens)
    assert [t for t, _ in got] == [t for t, _ in ref]
    assert all(abs(a[1] - b[1]) < 1e-12 for a, b in zip(got, ref))
    assert not math.isinf(got[0][1])
