"""ORACLE (test infrastructure only) — greedy, batched/pruned greedy, beam search.

* greedy_def: "we use greedy search in all submissions";
  argmax over raw logits — "remove the log_softmax in the output layer for
  greedy search" — ties to the lowest id (reading R13).  A
  sentence finishes on EOS or after cap_i = min(200, tgt_cap_i) generated
  tokens (reading R12).  Uses O-def (no cache).
  Pinned: == translate_fast (cached, batched, pruned) token for token;
  argmax(logits) == argmax(log_softmax(logits)).
* translate_fast: dynamic batches, cached decoding
   and batch pruning — "we prune the finished hypotheses in a
  batch during decoding" — with reading R18: a decision
  point after every ``prune_every`` steps; if #done >= max(1, ceil(rho B_live))
  (or all done) the live rows are compacted stably, new_to_old = ascending
  indices of the not-done rows.  Finished-but-unpruned rows keep computing and
  their tokens are ignored.  Pinned: outputs invariant to rho and to batching;
  == greedy_def.
* beam_search: "the search ends when any candidate predicts the EOS symbol,
  and there are no candidates with higher scores", reading R15:
  score = sum of log_softmax (no length penalty, R16); candidates (slot, v)
  ordered by (score desc, slot*V + v asc), first 2K kept; EOS candidates ranked
  < K are finalised; the first K non-EOS become the next active set; stop when
  fin is non-empty and max fin >= max active, or at the cap (actives finalised).
  Pinned: K >= V^T equals ``exhaustive_best`` (brute force); K = 1 == greedy;
  early stop on == off.
* beam_search_nbest: the N-best lists used for sequence-level KD ("we collected
  the 4-best list for each sentence"), reading R27: the finished
  list keeps the N best (score desc, ties -> earlier finalised); the search stops
  when N hypotheses are finished and the N-th best >= the best active (sound:
  scores never increase), or at the cap (actives finalised).  N = 1 is
  beam_search.  Pinned: K >= V^T equals ``exhaustive_nbest`` (brute force);
  early stop on == off; N = 1 == beam_search.
* ensemble_step_logprobs: the teacher ensemble ("a simple
  ensemble strategy"), reading R26: per step the members' next-token
  distributions are averaged, log p = logsumexp_m(log p_m) - log M (fairseq's
  ensemble).  Pinned: M copies of one model == that model; K >= V^T ensemble
  beam == brute force over the averaged distribution.
"""
from __future__ import annotations

import math

import numpy as np

from synth.config import BOS_ID, EOS_ID
from .nn import log_softmax
from .batching import plan_batches


def _cap(cfg, c):
    return int(min(cfg.max_tgt_len, int(c)))


# ------------------------------------------------------------------ greedy (def)
def greedy_def(model, src, cap: int, return_logits: bool = False):
    enc = model.encode_def(src)
    prefix = [BOS_ID]
    out, logits_all = [], []
    cap = _cap(model.cfg, cap)
    while True:
        logits = model.decoder_logits_def(enc, prefix)
        logits_all.append(logits)
        w = int(np.argmax(logits))
        out.append(w)
        prefix.append(w)
        if w == EOS_ID or len(out) == cap:
            break
    toks = out[:-1] if out[-1] == EOS_ID else out
    return (toks, np.array(logits_all)) if return_logits else toks


# ------------------------------------------------------ greedy (fast, batched)
def translate_fast(model, wl, max_tokens: int = 4096, max_sents: int = 512,
                   prune_every: int = 1, prune_ratio: float = 0.25, log: dict | None = None):
    """Greedy translation of a Workload; returns list of outputs in input order.

    ``log`` (optional dict) receives 'prunes': [(batch, step, new_to_old)],
    'gen_tokens', 'steps', 'batches', 'margins': per sentence, the top1 - top2
    logit gap at every generated position (which positions are margin-safe), and
    'scales': per sentence, max |logit| at every generated position (the FP32
    tolerance scale).  Logging only: no effect on the outputs.
    """
    cfg = model.cfg
    lens = wl.lengths()
    batches = plan_batches(lens, max_tokens, max_sents)
    outputs = [None] * wl.n
    prunes = []
    margins = [None] * wl.n
    scales = [None] * wl.n
    gen_tokens = 0
    steps = 0
    for bi, idx in enumerate(batches):
        srcs = [wl.sentence(i) for i in idx]
        caps = np.array([_cap(cfg, wl.caps[i]) for i in idx])
        enc, src_len = model.encode_batch(srcs)
        ckv = model.cross_kv(enc)
        B = len(idx)
        cache = model.new_cache(B, int(caps.max()))
        rows = np.arange(B)                 # live row -> batch slot
        tok = np.full(B, BOS_ID, dtype=np.int64)
        done = np.zeros(B, dtype=bool)
        gen = [[] for _ in range(B)]
        gaps = [[] for _ in range(B)]
        scl = [[] for _ in range(B)]
        t = 0
        while True:
            logits = model.decoder_step(tok, t, cache, ckv, src_len)
            nxt = np.argmax(logits, axis=1)
            top2 = np.partition(logits, -2, axis=1)[:, -2:]
            for r, s in enumerate(rows):
                if not done[r]:
                    gen[s].append(int(nxt[r]))
                    gaps[s].append(float(top2[r, 1] - top2[r, 0]))
                    scl[s].append(float(np.abs(logits[r]).max()))
                    if nxt[r] == EOS_ID or len(gen[s]) == caps[s]:
                        done[r] = True
            tok = nxt
            t += 1
            steps += 1
            if done.all():
                break
            if prune_ratio is not None and prune_ratio >= 0 and t % prune_every == 0:
                need = max(1, math.ceil(prune_ratio * len(rows)))
                if done.sum() >= need:
                    keep = np.nonzero(~done)[0]
                    prunes.append((bi, t - 1, keep.copy()))
                    rows, tok, done, src_len = rows[keep], tok[keep], done[keep], src_len[keep]
                    cache = [(K[keep], V[keep]) for K, V in cache]
                    ckv = [(K[keep], V[keep]) for K, V in ckv]
        for s, i in enumerate(idx):
            g = gen[s]
            gen_tokens += len(g)
            outputs[i] = g[:-1] if g and g[-1] == EOS_ID else g
            margins[i] = gaps[s]
            scales[i] = scl[s]
    if log is not None:
        log.update(prunes=prunes, gen_tokens=gen_tokens, steps=steps, batches=batches, margins=margins,
                   scales=scales)
    return outputs


# ----------------------------------------------------------------- beam search
def prefix_logprobs(model, enc_kv, src_len, prefixes):
    """log_softmax of next-token logits for each prefix (cached recompute)."""
    out = []
    for pre in prefixes:
        T = len(pre)
        cache = model.new_cache(1, T)
        for t in range(T):
            logits = model.decoder_step(np.array([pre[t]]), t, cache, enc_kv, src_len)
        out.append(log_softmax(logits[0]))
    return out


def beam_search(model, src, cap: int, K: int, early_stop: bool = True, step_logprobs=None):
    """Single-sentence beam search (reading R15).  Returns (tokens, score)."""
    return beam_search_nbest(model, src, cap, K, 1, early_stop, step_logprobs)[0]


def _strip(seq):
    toks = seq[1:]
    if toks and toks[-1] == EOS_ID:
        toks = toks[:-1]
    return toks


def beam_search_nbest(model, src, cap: int, K: int, nbest: int, early_stop: bool = True,
                      step_logprobs=None):
    """Beam search returning the ``nbest`` best finished hypotheses [(tokens, score)],
    best first (reading R27; nbest <= K)."""
    assert 1 <= nbest <= K
    cfg = model.cfg
    V = cfg.vocab_size
    cap = _cap(cfg, cap)
    enc, src_len = model.encode_batch([src])
    ckv = model.cross_kv(enc)
    if step_logprobs is None:
        def step_logprobs(prefixes):
            return prefix_logprobs(model, ckv, src_len, prefixes)
    active = [(0.0, [BOS_ID])]
    fin = []           # (score, tokens, order)
    order = 0
    for t in range(cap):
        lps = step_logprobs([h[1] for h in active])
        cand_s = np.concatenate([a[0] + lp for a, lp in zip(active, lps)])
        # order by (score desc, slot*V + v asc): lexsort keys are ascending, last key primary
        flat = np.arange(len(cand_s))
        sel = np.lexsort((flat, -cand_s))[:2 * K]
        new_active = []
        for rank, c in enumerate(sel):
            slot, v = divmod(int(c), V)
            sc = float(cand_s[c])
            if v == EOS_ID:
                if rank < K:
                    fin.append((sc, active[slot][1] + [v], order)); order += 1
            elif len(new_active) < K:
                new_active.append((sc, active[slot][1] + [v]))
        if t + 1 == cap:
            for sc, toks in new_active:
                fin.append((sc, toks, order)); order += 1
            break
        active = new_active
        if not active:
            break
        if early_stop and len(fin) >= nbest:
            nth = sorted(fin, key=lambda f: (-f[0], f[2]))[nbest - 1][0]
            if nth >= max(a[0] for a in active):
                break
    ranked = sorted(fin, key=lambda f: (-f[0], f[2]))[:nbest]
    return [(_strip(f[1]), f[0]) for f in ranked]


def exhaustive_nbest(model, src, cap: int, nbest: int, step_logprobs=None):
    """Brute force: the ``nbest`` highest-scoring complete sequences (EOS-terminated or
    cap-long) over every sequence of length <= cap; ties -> lexicographically smaller
    (token ids) first.  Returns [(tokens, score)]."""
    cfg = model.cfg
    cap = _cap(cfg, cap)
    if step_logprobs is None:
        enc, src_len = model.encode_batch([src])
        ckv = model.cross_kv(enc)

        def step_logprobs(prefixes):
            return prefix_logprobs(model, ckv, src_len, prefixes)
    done = []

    def rec(prefix, score):
        lp = step_logprobs([prefix])[0]
        for v in range(cfg.vocab_size):
            s = score + float(lp[v])
            seq = prefix + [v]
            if v == EOS_ID or len(seq) - 1 == cap:
                done.append((s, seq))
            else:
                rec(seq, s)

    rec([BOS_ID], 0.0)
    done.sort(key=lambda f: (-f[0], f[1]))
    return [(_strip(f[1]), f[0]) for f in done[:nbest]]


def ensemble_step_logprobs(models, srcs_or_src):
    """Step function for beam_search(_nbest): the members' log-probabilities averaged in
    probability space, logsumexp_m(lp_m) - log M (reading R26).  ``models`` are
    OracleModel instances with equal vocabularies; the source is encoded by each."""
    src = srcs_or_src
    ctx = []
    for mdl in models:
        enc, src_len = mdl.encode_batch([src])
        ctx.append((mdl, mdl.cross_kv(enc), src_len))

    def step(prefixes):
        lps = np.stack([prefix_logprobs(mdl, ckv, sl, prefixes) for mdl, ckv, sl in ctx])
        mx = lps.max(axis=0)
        return mx + np.log(np.exp(lps - mx).sum(axis=0)) - math.log(len(models))
    return step


def exhaustive_best(model, src, cap: int):
    """Brute force over every sequence of length <= cap (EOS-terminated or cap-long)."""
    cfg = model.cfg
    cap = _cap(cfg, cap)
    enc, src_len = model.encode_batch([src])
    ckv = model.cross_kv(enc)
    best = (-math.inf, None)

    def rec(prefix, score):
        nonlocal best
        lp = prefix_logprobs(model, ckv, src_len, [prefix])[0]
        for v in range(cfg.vocab_size):
            s = score + float(lp[v])
            seq = prefix + [v]
            if v == EOS_ID or len(seq) - 1 == cap:
                if s > best[0]:
                    best = (s, seq[1:])
            else:
                rec(seq, s)

    rec([BOS_ID], 0.0)
    toks = best[1]
    if toks and toks[-1] == EOS_ID:
        toks = toks[:-1]
    return toks, best[0]
