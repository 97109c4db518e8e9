"""ORACLE (test infrastructure only) — the text pipeline of §8(f) row f3.

"the data was tokenized, and jointly byte pair encoded with 32K merge operations using a
shared vocabulary.  After decoding, we removed the BPE separators", with the
C++ subword tool of PAPER.md:141 (fastBPE conventions).  Readings (R28, from the SPEC's
text-pipeline module): input lines are pretokenised (split on ASCII whitespace); a word
starts as its characters (Unicode code points); repeatedly the adjacent pair of lowest
merge rank is merged at every non-overlapping occurrence, left to right, until no pair is
in the table; every subword but the word-final one carries the separator "@@".  Removal
joins tokens with single spaces and deletes every "@@ ".  Vocabulary: reserved PAD, UNK,
BOS, EOS = 0..3, file token i -> id 4 + i; encoding maps unknown tokens to UNK and appends
EOS; decoding stops at EOS and skips reserved ids.

Pinned by the worked examples of the SPEC (tests/golden/bpe_examples.txt) and the
round-trip property bpe_remove(bpe_apply(L)) == whitespace-normalised L.
"""
from __future__ import annotations

import re

PAD, UNK, BOS, EOS = 0, 1, 2, 3
_WS = re.compile(r"[ \t\n\r\x0b\x0c]+")   # ASCII whitespace (pretokenised input)
SEP = "@@"


def load_merges(text: str):
    """Merge table: pair -> rank (line index among merge lines; '#version' lines skipped)."""
    ranks = {}
    r = 0
    for ln, line in enumerate(text.split("\n"), 1):
        if not line.strip() or line.startswith("#version"):
            continue
        parts = [x for x in _WS.split(line) if x]
        if len(parts) != 2:
            raise ValueError(f"merges line {ln}: expected two symbols")
        pair = (parts[0], parts[1])
        if pair in ranks:
            raise ValueError(f"merges line {ln}: duplicate pair")
        ranks[pair] = r
        r += 1
    return ranks


def load_vocab(text: str):
    tok2id = {}
    for ln, line in enumerate(text.split("\n"), 1):
        tok = line.strip(" \t\r")
        if not tok:
            continue
        if tok in tok2id:
            raise ValueError(f"vocab line {ln}: duplicate token")
        tok2id[tok] = 4 + len(tok2id)
    id2tok = {i: t for t, i in tok2id.items()}
    return tok2id, id2tok


def bpe_word(word: str, ranks):
    sym = list(word)
    while len(sym) > 1:
        best = None
        for i in range(len(sym) - 1):
            r = ranks.get((sym[i], sym[i + 1]))
            if r is not None and (best is None or r < best):
                best = r
        if best is None:
            break
        out, i = [], 0
        while i < len(sym):
            if i + 1 < len(sym) and ranks.get((sym[i], sym[i + 1])) == best:
                out.append(sym[i] + sym[i + 1])
                i += 2
            else:
                out.append(sym[i])
                i += 1
        sym = out
    return [s + SEP for s in sym[:-1]] + sym[-1:]


def bpe_apply(line: str, ranks):
    toks = []
    for w in _WS.split(line):
        if w:
            toks.extend(bpe_word(w, ranks))
    return toks


def bpe_remove(tokens):
    return " ".join(tokens).replace(SEP + " ", "")


def encode_ids(tokens, tok2id):
    return [tok2id.get(t, UNK) for t in tokens] + [EOS]


def decode_ids(ids, id2tok, size):
    out = []
    for i in ids:
        if i < 0 or i >= size:
            raise ValueError(f"id {i} out of range")
        if i == EOS:
            break
        if i < 4:
            continue
        out.append(id2tok[i])
    return out
