"""-m gpu tests of the C-ABI boundary (include/nmt.h): the memory pool sized at
load, nmt_batch_free, caller-mask pruning, step-drivable beam search
(d_parent / d_score), source truncation in the translate drivers, per-call device timing."""
import numpy as np
import pytest
import torch

from synth import tiny_workload, newstest_like, random_tokens, BOS_ID, EOS_ID
from gpu_common import weights, oracle_model, gpu_model, logits_close, pad_batch

pytestmark = pytest.mark.gpu


def test_workspaces_allocated_at_load_and_flat():
    """Every arena is allocated by nmt_load_weights (limits.n_workspaces): translate never
    calls cudaMalloc — arena_system_allocs is the same after a second identical pass (the
    SPEC's pool-reuse check, S:545 analog) and n_workers above the pool is refused."""
    from paper_2109_08008_b200.nmt import NmtError
    wl = newstest_like(200, 32000, start=3000)
    gm = gpu_model("student-6-1", "fp16", max_tokens=1024, max_sents=64, workspaces=3)
    _, st1 = gm.translate(wl.ids, wl.off, caps=wl.caps, workers=3)
    _, st2 = gm.translate(wl.ids, wl.off, caps=wl.caps, workers=3)
    # weights + LN-folded weights + (device arena + pinned staging) per workspace
    assert st1["arena_system_allocs"] == st2["arena_system_allocs"] == 2 + 2 * 3
    assert st1["ms_encode"] > 0 and st1["ms_decode"] > 0
    with pytest.raises(NmtError) as e:
        gm.translate(wl.ids, wl.off, caps=wl.caps, workers=4)
    assert e.value.code == 1
    d_ids = torch.from_numpy(wl.ids).cuda()
    d_out = torch.zeros(wl.n, gm.Tmax, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(wl.n, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        st3 = gm.translate_device(d_ids, wl.off, d_out, d_len, caps=wl.caps, workers=2)
    torch.cuda.synchronize()
    assert st3["arena_system_allocs"] == st1["arena_system_allocs"]


def test_batch_free_invalidates_handle():
    from paper_2109_08008_b200.nmt import NmtError
    wl = tiny_workload(n=4)
    gm = gpu_model("tiny", "fp32", max_tokens=256, max_sents=8, max_tgt_len=32)
    src, lens = pad_batch([wl.sentence(i) for i in range(wl.n)])
    b = gm.encode(torch.from_numpy(src).cuda(), lens)
    h = b.h
    b.free()
    b.h = h   # a stale handle is rejected, not used
    with pytest.raises(NmtError) as e:
        b.decode_step(n_live=wl.n)
    assert e.value.code == 1
    b.h = None
    b2 = gm.encode(torch.from_numpy(src).cuda(), lens)   # the arena is reusable
    assert b2.live() == wl.n


def test_prune_keep_mask_matches_oracle():
    """nmt_prune_batch with the caller's keep mask (greedy): the map is the stable compaction
    of the mask, and the surviving rows continue exactly as the oracle's sentences do
    (teacher-forced FP32 logits within 1e-4) — removing rows changes nothing for the others
    (PAPER.md:104-105)."""
    wl = newstest_like(40, 1000, start=10)
    cfg, _ = weights("tiny")
    om = oracle_model("tiny")
    gm = gpu_model("tiny", "fp32", max_tokens=4096, max_sents=64, max_tgt_len=32)
    srcs = [wl.sentence(i)[-16:] for i in range(wl.n)]
    srcs = [np.concatenate([s[:-1], [EOS_ID]]) if s[-1] != EOS_ID else s for s in srcs]
    src, lens = pad_batch(srcs)
    b = gm.encode(torch.from_numpy(src).cuda(), lens)
    enc, sl = om.encode_batch([list(s) for s in srcs])
    ckv = om.cross_kv(enc)
    T = 6
    forced = np.concatenate([np.full((wl.n, 1), BOS_ID), random_tokens(wl.n, T - 1, 1000, seed=3)], 1)
    cache = om.new_cache(wl.n, T)
    rows = np.arange(wl.n)
    rng = np.random.default_rng(0)
    for t in range(T):
        prev = torch.from_numpy(forced[rows, t].astype(np.int32)).cuda()
        r = b.decode_step(prev=prev, logits=True, n_live=len(rows))
        lo = om.decoder_step(forced[rows, t], t, cache, ckv, sl)
        ok, worst = logits_close(r["logits"].double().cpu().numpy(), lo, "fp32")
        assert ok, (t, worst)
        assert (r["parent"].cpu().numpy() == np.arange(len(rows))).all()
        keep = (rng.random(len(rows)) > 0.3).astype(np.uint8)
        keep[0] = 1
        n, m = b.prune(keep=torch.from_numpy(keep).cuda())
        kk = np.flatnonzero(keep)
        assert n == len(kk)
        assert m.cpu().numpy()[:n].tolist() == kk.tolist()
        assert (m.cpu().numpy()[n:] == -1).all()
        rows = rows[kk]
        cache = [(K[kk], V[kk]) for K, V in cache]
        ckv = [(K[kk], V[kk]) for K, V in ckv]
        sl = sl[kk]


@pytest.mark.parametrize("ratio", [0.25, -1.0])
def test_beam_step_drivable(ratio):
    """Beam search driven step by step through the C ABI: after each
    nmt_decode_step the rows' (parent, next, score) rebuild every live hypothesis; each
    reported score equals the FP64 oracle's sum of log-probabilities of that hypothesis, and
    the batch results equal nmt_translate's beam output."""
    from gpu_common import oracle_step_logprobs, seq_logprob
    K = 4
    wl = tiny_workload(n=6, seed=11, max_cap=10)
    om = oracle_model("tiny", 3.0)
    gm = gpu_model("tiny", "fp32", 3.0, max_tokens=256, max_sents=8, max_tgt_len=32, beam=K)
    order = np.argsort(-wl.lengths(), kind="stable")
    srcs = [wl.sentence(i) for i in order]
    caps = wl.caps[order]
    src, lens = pad_batch(srcs)
    b = gm.encode(torch.from_numpy(src).cuda(), lens, tgt_cap=caps, beam=K)
    slp = [oracle_step_logprobs(om, s) for s in srcs]
    hyps = [[] for _ in range(wl.n * K)]     # tokens of the hypothesis in each live row
    sent = np.repeat(np.arange(wl.n), K)     # sentence of each live row
    n = wl.n * K
    checked = 0
    for t in range(32):
        r = b.decode_step(n_live=n)
        par = r["parent"].cpu().numpy()
        nxt = r["next"].cpu().numpy()
        sc = r["score"].cpu().numpy()
        dn = r["done"].cpu().numpy()
        new = []
        for row in range(n):
            if par[row] >= 0:
                assert sent[par[row]] == sent[row]   # a hypothesis stays in its sentence
                h = hyps[par[row]] + [int(nxt[row])]
                if np.isfinite(sc[row]):
                    ref = seq_logprob(slp[sent[row]], h, len(h))   # cap = len: no EOS, an open prefix
                    assert abs(sc[row] - ref) <= 1e-4 * max(1.0, abs(ref)), (t, row, h)
                    checked += 1
                new.append(h)
            else:
                assert dn[row] or not np.isfinite(sc[row])
                new.append(hyps[row])
        hyps = new
        n_new, m = b.prune(ratio=ratio)
        m = m.cpu().numpy()[:n_new]
        hyps = [hyps[i] for i in m]
        sent = sent[m]
        n = n_new
        if n == 0:
            break
    assert n == 0 and checked > 0
    ids, ln = b.results()
    out_step = [ids[j, :ln[j]].tolist() for j in range(wl.n)]
    out_step = [o[:-1] if o and o[-1] == EOS_ID else o for o in out_step]
    full, _ = gm.translate(wl.ids[np.concatenate([np.arange(wl.off[i], wl.off[i + 1]) for i in order])],
                           np.concatenate([[0], np.cumsum(wl.lengths()[order])]), caps=caps,
                           max_tokens=256, max_sents=8, beam=K, prune_ratio=ratio)
    assert out_step == full


def test_truncation_long_source():
    """ADVICE r1 / SURVEY §8(b): translate truncates a source longer than max_src_len to
    max_src_len - 1 tokens + EOS (counted) instead of rejecting the whole run; the output
    equals translating the truncated source.  nmt_encode still rejects (NMT_E_INPUT)."""
    from paper_2109_08008_b200.nmt import NmtError
    r = np.random.default_rng(4)
    long = np.concatenate([r.integers(4, 1000, 299), [EOS_ID]]).astype(np.int32)
    short = np.array([5, 6, 7, EOS_ID], dtype=np.int32)
    cut = np.concatenate([long[:119], [EOS_ID]]).astype(np.int32)
    gm = gpu_model("tiny", "fp32", max_tokens=512, max_sents=8, max_tgt_len=32)

    def run(srcs, device=False):
        ids = np.concatenate(srcs)
        off = np.concatenate([[0], np.cumsum([len(s) for s in srcs])]).astype(np.int64)
        caps = np.full(len(srcs), 12, dtype=np.int32)
        if not device:
            return gm.translate(ids, off, caps=caps)
        d_out = torch.zeros(len(srcs), gm.Tmax, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(len(srcs), dtype=torch.int32, device="cuda")
        st = gm.translate_device(torch.from_numpy(ids).cuda(), off, d_out, d_len, caps=caps)
        torch.cuda.synchronize()
        o = [d_out[i, :d_len[i]].tolist() for i in range(len(srcs))]
        return [x[:-1] if x and x[-1] == EOS_ID else x for x in o], st
    a, sa = run([short, long, short])
    b, sb = run([short, cut, short])
    assert a == b and sa["truncated"] == 1 and sb["truncated"] == 0
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        c, sc = run([short, long, short], device=True)
    assert c == a and sc["truncated"] == 1
    with pytest.raises(NmtError) as e:
        gm.encode(torch.from_numpy(long[None, :]).cuda(), [300])
    assert e.value.code in (2, 3)
