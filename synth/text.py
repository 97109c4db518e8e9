"""Seeded synthetic text artifacts for the text pipeline (§8(f) row f3): a merge table, a
shared vocabulary file and pretokenised lines.  Random tables only — no BPE arithmetic
(both the oracle and the library apply the merges themselves).

The paper's tables come from 32K merges learned on WMT data, which is not
available here; the synthetic table has the same form (ordered symbol pairs, rank = line).
"""
from __future__ import annotations

import numpy as np

TEXT_SEED = 31


def synthetic_bpe(n_merges: int = 300, alphabet: str = "abcdefghijklmnopqrstuvwxyzäöüß",
                  seed: int = TEXT_SEED, pad_to: int = 0):
    """Returns (merges_text, vocab_text, symbols).  Merge i joins two symbols that exist
    before it (characters or earlier merge results); the vocabulary lists every symbol
    both bare and with the "@@" separator (fastBPE's shared vocabulary form)."""
    rng = np.random.default_rng(seed)
    symbols = list(alphabet)
    pairs, seen = [], set()
    while len(pairs) < n_merges:
        a = symbols[int(rng.integers(len(symbols)))]
        b = symbols[int(rng.integers(len(symbols)))]
        if (a, b) in seen or len(a) + len(b) > 8:
            continue
        seen.add((a, b))
        pairs.append((a, b))
        if a + b not in symbols:
            symbols.append(a + b)
    merges_text = "#version 0.2\n" + "\n".join(f"{a} {b}" for a, b in pairs) + "\n"
    vocab = []
    for s in symbols:
        vocab += [s, s + "@@"]
    if pad_to:   # fill up to a model vocabulary (pad_to = ModelConfig.vocab_size)
        vocab += [f"<unused{i}>" for i in range(pad_to - 4 - len(vocab))]
    vocab_text = "\n".join(vocab) + "\n"
    return merges_text, vocab_text, symbols


def synthetic_lines(n: int, symbols, seed: int = TEXT_SEED + 1, max_words: int = 12,
                    oov_rate: float = 0.02):
    """Pretokenised lines of words built from random symbol sequences (some characters
    outside the alphabet give unknown-token paths); irregular whitespace on purpose."""
    rng = np.random.default_rng(seed)
    lines = []
    for _ in range(n):
        words = []
        for _ in range(int(rng.integers(1, max_words + 1))):
            w = "".join(symbols[int(rng.integers(len(symbols)))] for _ in range(int(rng.integers(1, 4))))
            if rng.random() < oov_rate:
                w += "#"
            words.append(w)
        sep = "  " if rng.random() < 0.2 else " "
        lines.append(sep.join(words) + (" " if rng.random() < 0.1 else ""))
    return lines
