"""§8(f) row f3 — the text pipeline ("jointly byte pair encoded with 32K merge
operations using a shared vocabulary ... we removed the BPE separators", PAPER.md:141 the
C++ subword tool; reading R28).  The codec is host code in libnmt.so, so these run on CPU:

* the oracle (oracle/text.py) against the worked examples of tests/golden/bpe_examples.txt
  and the round-trip property remove(apply(L)) == whitespace-normalised L;
* the library codec (nmt_text_*) against the oracle, id for id, on seeded synthetic lines
  (UTF-8 letters, unknown characters, irregular whitespace), single- and multi-threaded;
* decoding: EOS stops, reserved ids are skipped, separators removed; error contracts."""
import os

import numpy as np
import pytest

from oracle.text import (load_merges, load_vocab, bpe_apply, bpe_remove, encode_ids,
                         decode_ids, EOS)
from synth.text import synthetic_bpe, synthetic_lines

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    rows = []
    for line in open(os.path.join(HERE, "golden", "bpe_examples.txt"), encoding="utf-8"):
        if line.startswith("#") or not line.strip():
            continue
        kind, merges, inp, exp = [x.strip() for x in line.split("|")]
        merges = "\n".join(m.strip() for m in merges.split(";") if m.strip())
        rows.append((kind, merges, inp, exp))
    return rows


def _codec(vocab_text, merges_text):
    from paper_2109_08008_b200 import TextCodec
    return TextCodec(vocab_text, merges_text)


@pytest.mark.parametrize("row", _golden())
def test_golden_examples(row):
    kind, merges, inp, exp = row
    if kind == "apply":
        toks = bpe_apply(inp, load_merges(merges))
        assert toks == exp.split()
        # the library codec gives the same tokens (vocabulary = the expected tokens)
        vocab = "\n".join(exp.split())
        tok2id, id2tok = load_vocab(vocab)
        c = _codec(vocab, merges)
        ids, off = c.encode([inp])
        assert [id2tok[i] for i in ids[:-1]] == exp.split() and ids[-1] == EOS
    else:
        assert bpe_remove(inp.split()) == exp


def test_oracle_round_trip():
    m, v, sym = synthetic_bpe()
    ranks = load_merges(m)
    for line in synthetic_lines(200, sym):
        assert bpe_remove(bpe_apply(line, ranks)) == " ".join(line.split())


@pytest.mark.parametrize("threads", [1, 4])
def test_library_encode_matches_oracle(threads):
    m, v, sym = synthetic_bpe()
    ranks = load_merges(m)
    tok2id, _ = load_vocab(v)
    lines = synthetic_lines(400, sym)
    c = _codec(v, m)
    assert c.vocab_size == 4 + len(tok2id)
    ids, off = c.encode(lines, threads=threads)
    assert len(off) == len(lines) + 1
    for i, line in enumerate(lines):
        assert ids[off[i]:off[i + 1]].tolist() == encode_ids(bpe_apply(line, ranks), tok2id)


def test_library_decode_matches_oracle():
    m, v, sym = synthetic_bpe()
    tok2id, id2tok = load_vocab(v)
    V = 4 + len(tok2id)
    rng = np.random.default_rng(5)
    seqs = []
    for _ in range(200):
        s = rng.integers(0, V, size=int(rng.integers(0, 20))).tolist()
        if rng.random() < 0.5:
            s.insert(int(rng.integers(0, len(s) + 1)), EOS)
        seqs.append(s)
    off = np.cumsum([0] + [len(s) for s in seqs])
    c = _codec(v, m)
    got = c.decode(np.array(sum(seqs, []), dtype=np.int32), off)
    assert got == [bpe_remove(decode_ids(s, id2tok, V)) for s in seqs]


def test_library_round_trip_in_vocab():
    m, v, sym = synthetic_bpe()
    lines = [ln for ln in synthetic_lines(300, sym, oov_rate=0.0)]
    c = _codec(v, m)
    ids, off = c.encode(lines)
    assert c.decode(ids, off) == [" ".join(ln.split()) for ln in lines]


def test_unknown_tokens_and_reserved():
    m, v, sym = synthetic_bpe()
    c = _codec(v, m)
    ids, off = c.encode(["ab#c", "", "zz"])
    assert 1 in ids[off[0]:off[1]].tolist()              # '#' has no vocabulary entry -> UNK
    assert ids[off[1]:off[2]].tolist() == [EOS]           # an empty line is just EOS
    # decoding never emits PAD / UNK / BOS and stops at EOS
    assert c.decode(np.array([0, 1, 2, 3, 4], dtype=np.int32), np.array([0, 5])) == [""]


def test_error_contracts():
    from paper_2109_08008_b200 import NmtError
    with pytest.raises(NmtError, match="line 3"):
        _codec("a\nb\n", "a b\nc d\na b\n")                # duplicate pair
    with pytest.raises(NmtError, match="line 2"):
        _codec("a\na\n", "")                               # duplicate token
    with pytest.raises(NmtError, match="line 1"):
        _codec("a\n", "a b c\n")                           # malformed merge
    c = _codec("a\n", "")
    with pytest.raises(NmtError):
        c.decode(np.array([9], dtype=np.int32), np.array([0, 1]))
