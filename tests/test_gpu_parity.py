"""-m gpu parity tests: the CUDA path through the C ABI vs the FP64 oracle on the same
seeded inputs (tiny C1 in full; 6-1 / 35-1 on subsets spanning several tiles, the
RPR clip boundary and ragged tails).  FP32 mode within 1e-4 relative, FP16 within
2e-2 absolute; greedy tokens bit-exact on margin-safe positions; prune maps bit-exact."""
import numpy as np
import pytest
import torch

from synth import tiny_workload, newstest_like, random_tokens, BOS_ID, PRESETS
from gpu_common import (TOL, weights, oracle_model, gpu_model, logits_close, margin_safe, pad_batch,
                        safe_prefix_len, greedy_valid, beam_valid, oracle_step_logprobs)

pytestmark = pytest.mark.gpu

PRECS = ["fp32", "fp16"]


# ------------------------------------------------------------------ GEMM units
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,N,K", [(1, 64, 64), (3, 512, 512), (148, 1536, 512), (300, 2048, 512),
                                   (129, 512, 2048), (4096, 512, 512), (77, 1000, 64), (512, 32000, 512),
                                   (4099, 512, 2048)])
def test_gemm_unit(prec, M, N, K):
    from paper_2109_08008_b200 import dev_gemm
    g = torch.Generator().manual_seed(M * 7 + N + K)
    dt = torch.float16 if prec == "fp16" else torch.float32
    A = (torch.randn(M, K, generator=g) / 2).to(dt)
    B = (torch.randn(N, K, generator=g) / K ** 0.5).to(dt)
    bias = (torch.randn(N, generator=g) * 0.1).to(dt)
    R = torch.randn(M, N, generator=g).to(dt)
    ref = A.double() @ B.double().T + bias.double() + R.double()
    for relu in (False, True):
        r = ref.clamp_min(0) if relu else ref
        out = dev_gemm(A.cuda(), B.cuda(), bias.cuda(), R.cuda(), relu=relu).double().cpu()
        if prec == "fp32":
            tol = 1e-4 * max(1.0, float(r.abs().max()))
            assert float((out - r).abs().max()) <= tol
        else:  # FP16 output rounding (2^-11 relative) + FP32 accumulation
            assert float(((out - r).abs() / (r.abs() + 1)).max()) <= 2e-3
    out = dev_gemm(A.cuda(), B.cuda()).double().cpu()
    r = A.double() @ B.double().T
    assert float(((out - r).abs() / (r.abs() + 1)).max()) <= (1e-5 if prec == "fp32" else 2e-3)


@pytest.mark.parametrize("M,N,K", [(1, 1536, 512), (148, 512, 512), (148, 2048, 512), (300, 512, 2048),
                                   (512, 1536, 512), (37, 64, 64), (9, 256, 64)])
def test_gemm_decode_unit(M, N, K):
    """The decode-step GEMM configuration (gemm_tc.cu decode_config): correct, deterministic
    and batch invariant (a row's result does not depend on the other rows)."""
    from paper_2109_08008_b200 import dev_gemm_decode, dev_gemm
    g = torch.Generator().manual_seed(M + 3 * N + K)
    A = (torch.randn(M, K, generator=g) / 2).half()
    B = (torch.randn(N, K, generator=g) / K ** 0.5).half()
    bias = (torch.randn(N, generator=g) * 0.1).half()
    R = torch.randn(M, N, generator=g).half()
    ref = A.double() @ B.double().T + bias.double() + R.double()
    for relu in (False, True):
        r = ref.clamp_min(0) if relu else ref
        out = dev_gemm_decode(A.cuda(), B.cuda(), bias.cuda(), R.cuda(), relu=relu)
        assert float(((out.double().cpu() - r).abs() / (r.abs() + 1)).max()) <= 2e-3
        again = dev_gemm_decode(A.cuda(), B.cuda(), bias.cuda(), R.cuda(), relu=relu)
        assert torch.equal(out, again)                      # deterministic reduction order
    # rows are independent of the other rows (batch invariance of the split policy)
    full = dev_gemm_decode(A.cuda(), B.cuda(), bias.cuda(), R.cuda())
    part = dev_gemm_decode(A[: max(1, M // 3)].cuda(), B.cuda(), bias.cuda(), R[: max(1, M // 3)].cuda())
    assert torch.equal(full[: max(1, M // 3)], part)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("M,N", [(1, 1000), (148, 32000), (513, 32000), (5, 8)])
def test_gemm_argmax_unit(prec, M, N):
    from paper_2109_08008_b200 import dev_gemm_argmax
    K = 64 if N < 100 else 512
    g = torch.Generator().manual_seed(M + N)
    dt = torch.float16 if prec == "fp16" else torch.float32
    A = torch.randn(M, K, generator=g).to(dt)
    B = (torch.randn(N, K, generator=g) / K ** 0.5).to(dt)
    nxt, lg = dev_gemm_argmax(A.cuda(), B.cuda(), logits=True)
    ref = (A.double() @ B.double().T).numpy()
    ok, worst = logits_close(lg.double().cpu().numpy(), ref, prec)
    assert ok, worst
    # the fused argmax equals argmax of the kernel's own FP32 logits, ties -> lowest id
    lgn = lg.cpu().numpy()
    assert (nxt.cpu().numpy() == np.argmax(lgn, axis=1)).all()
    safe = margin_safe(ref, prec)
    assert (nxt.cpu().numpy()[safe] == np.argmax(ref, axis=1)[safe]).all()


def test_argmax_ties_lowest_id():
    from paper_2109_08008_b200 import dev_gemm_argmax
    A = torch.ones(4, 64, dtype=torch.float16, device="cuda")
    B = torch.zeros(1000, 64, dtype=torch.float16, device="cuda")
    B[[7, 300, 999]] = 1.0        # three equal maxima
    assert (dev_gemm_argmax(A, B).cpu() == 7).all()


# ------------------------------------------------------------------ model parity
# ------------------------------------------------------------------ encoder attention unit
@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("S,lens", [(5, [5, 2]), (16, [16, 9, 1]), (23, [23, 17, 8, 23]),
                                    (32, [32, 31, 30]), (41, [41, 9]), (77, [77, 60]),
                                    (120, [120, 64, 7])])
def test_attn_encoder_unit(prec, S, lens):
    """Encoder RPR self-attention through nmt_dev_attn_encoder vs the oracle's plain double
    loop (oracle.nn.rpr_attention_loops, Shaw et al. keys and values):
    every padded length class of the FP16 TMA pipeline (SP = 16..128), ragged lengths,
    sentences shorter than the clip distance, query rows >= len written 0."""
    from oracle.nn import rpr_attention_loops
    from paper_2109_08008_b200 import dev_attn_encoder
    rng = np.random.default_rng(1000 + S)
    B, d, H, kc = len(lens), 512, 8, 8
    dt = torch.float16 if prec == "fp16" else torch.float32
    qkv = torch.from_numpy(rng.standard_normal((B * S, 3 * d))).to(dt)
    relk = torch.from_numpy(0.5 * rng.standard_normal((2 * kc + 1, d // H))).to(dt)
    relv = torch.from_numpy(0.5 * rng.standard_normal((2 * kc + 1, d // H))).to(dt)
    ln = torch.tensor(lens, dtype=torch.int32)
    out = dev_attn_encoder(qkv.cuda(), ln.cuda(), relk.cuda(), relv.cuda(), B, S, H, kc)
    g = out.float().cpu().numpy()
    x = qkv.double().numpy()
    ak, av = relk.double().numpy(), relv.double().numpy()
    for b, n in enumerate(lens):
        rows = x[b * S:b * S + n]
        ref = rpr_attention_loops(rows[:, :d], rows[:, d:2 * d], rows[:, 2 * d:], ak, av, H, kc,
                                  lambda i, j: (True, i))
        got = g[b * S:(b + 1) * S]
        tol = 1e-4 if prec == "fp32" else 1e-2
        assert np.abs(got[:n] - ref).max() <= tol * max(1.0, np.abs(ref).max()), (b, n)
        assert not np.any(got[n:]), "padding query rows must be zero"


@pytest.mark.parametrize("pattern", ["random", "block37", "block18"])
@pytest.mark.parametrize("S", [32, 48, 64])
def test_attn_encoder_slot_handoff(S, pattern):
    """FP16 encoder attention at batch scale with sentence lengths mixing 1 and S: the
    persistent CTAs walk ~50 (sentence, head) items each through a ring of shared-memory
    slots, units round robin over the consumer warps, so warps whose items are short run
    rounds ahead of the warps on long items -- the slot hand-off must still give every unit
    its own item (csrc/attention_tc.cu, wait_issued).  The batch result is bit-identical to
    launches of 30 sentences (at most one item per CTA: no slot reuse) and across repeats,
    padding rows are zero, and sampled sentences match the oracle's double loop.  block37 /
    block18 alternate long and short runs of sentences so that a CTA's consecutive items
    (G = 296 / 148 CTAs apart, 8 heads) alternate long and short."""
    from oracle.nn import rpr_attention_loops
    from paper_2109_08008_b200 import dev_attn_encoder
    rng = np.random.default_rng(77 + S)
    B, d, H, kc = 2000, 512, 8, 8
    if pattern == "random":
        lens = np.where(rng.random(B) < 0.5, 1, S).astype(np.int32)
        mid = rng.random(B) < 0.2
        lens[mid] = rng.integers(1, S + 1, size=int(mid.sum()))
    else:
        blk = int(pattern[5:])
        lens = np.where((np.arange(B) // blk) % 2 == 1, S, 1).astype(np.int32)
    qkv = torch.from_numpy(rng.standard_normal((B * S, 3 * d))).to(torch.float16).cuda()
    relk = torch.from_numpy(0.5 * rng.standard_normal((2 * kc + 1, d // H))).to(torch.float16).cuda()
    relv = torch.from_numpy(0.5 * rng.standard_normal((2 * kc + 1, d // H))).to(torch.float16).cuda()
    ln = torch.from_numpy(lens).cuda()
    outs = [dev_attn_encoder(qkv, ln, relk, relv, B, S, H, kc) for _ in range(3)]
    ref = torch.cat([dev_attn_encoder(qkv[b0 * S:min(B, b0 + 30) * S].contiguous(), ln[b0:b0 + 30].contiguous(),
                                      relk, relv, min(30, B - b0), S, H, kc) for b0 in range(0, B, 30)])
    torch.cuda.synchronize()
    for o in outs:
        bad = (o != ref).reshape(B, -1).any(1).nonzero().flatten().tolist()
        assert not bad, (len(bad), bad[:8])
    g = outs[0].float().cpu().numpy().reshape(B, S, d)
    pad = np.arange(S)[None, :] >= lens[:, None]
    assert not np.any(g[pad]), "padding query rows must be zero"
    x = qkv.double().cpu().numpy()
    ak, av = relk.double().cpu().numpy(), relv.double().cpu().numpy()
    for b in rng.choice(np.nonzero(lens > 1)[0], 8, replace=False):
        n = int(lens[b])
        rows = x[b * S:b * S + n]
        want = rpr_attention_loops(rows[:, :d], rows[:, d:2 * d], rows[:, 2 * d:], ak, av, H, kc,
                                   lambda i, j: (True, i))
        assert np.abs(g[b, :n] - want).max() <= 1e-2 * max(1.0, np.abs(want).max()), (b, n)


def _teacher_forced(name, prec, srcs, forced, eos_boost=1.0):
    """Run encoder + forced decode on GPU and oracle; compare encoder out and logits."""
    cfg, _ = weights(name, eos_boost)
    om = oracle_model(name, eos_boost)
    gm = gpu_model(name, prec, eos_boost, max_tokens=4096, max_sents=64, max_tgt_len=64)
    src, lens = pad_batch(srcs)
    batch = gm.encode(torch.from_numpy(src).cuda(), lens)
    enc_o, lens_o = om.encode_batch(srcs)
    enc_g = batch.encoder_output().cpu().numpy()
    B, T = forced.shape
    for b in range(B):   # compare valid positions only (padding rows are unused)
        ok, worst = logits_close(enc_g[b, :lens[b]], enc_o[b, :lens[b]], prec)
        assert ok, ("encoder", b, worst)
    ckv = om.cross_kv(enc_o)
    cache = om.new_cache(B, T)
    worst_all = 0.0
    for t in range(T):
        prev = torch.from_numpy(forced[:, t].astype(np.int32)).cuda()
        r = batch.decode_step(prev=prev, logits=True, n_live=B)
        lo = om.decoder_step(forced[:, t], t, cache, ckv, lens_o)
        lg = r["logits"].double().cpu().numpy()
        ok, worst = logits_close(lg, lo, prec)
        worst_all = max(worst_all, worst)
        assert ok, ("step", t, worst)
        safe = margin_safe(lo, prec)
        assert (r["next"].cpu().numpy()[safe] == np.argmax(lo, 1)[safe]).all(), ("argmax", t)
        n, _ = batch.prune(ratio=-1.0, want_map=False)
        assert n == B
    return worst_all


@pytest.mark.parametrize("prec", PRECS)
def test_tiny_teacher_forced(prec):
    wl = tiny_workload()
    srcs = [wl.sentence(i) for i in range(wl.n)]
    T = 20   # spans the RPR clip boundary t = 8/9
    forced = np.concatenate([np.full((wl.n, 1), BOS_ID), random_tokens(wl.n, T - 1, 1000)], 1)
    _teacher_forced("tiny", prec, srcs, forced)


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["student-6-1", "student-35-1", "student-9-1-tiny"])
def test_base_teacher_forced(prec, name):
    wl = newstest_like(24, 32000)
    srcs = [wl.sentence(i) for i in range(wl.n)]
    T = 12
    forced = np.concatenate([np.full((wl.n, 1), BOS_ID), random_tokens(wl.n, T - 1, 32000, seed=5)], 1)
    _teacher_forced(name, prec, srcs, forced)


def _free_running(name, prec, wl, eos_boost, max_tokens=4096, max_sents=512, ratio=0.25):
    from oracle import translate_fast
    om = oracle_model(name, eos_boost)
    log = {}
    ref = translate_fast(om, wl, max_tokens, max_sents, prune_ratio=ratio, log=log)
    gm = gpu_model(name, prec, eos_boost, max_tokens=max_tokens, max_sents=max_sents)
    out, st = gm.translate(wl.ids, wl.off, caps=wl.caps, max_tokens=max_tokens, max_sents=max_sents,
                           prune_ratio=ratio)
    n_cmp = 0
    full = True
    for i in range(wl.n):
        g, o = out[i], ref[i]
        # bit-exact up to the first margin-unsafe position (SURVEY §8(c) tokens rule) ...
        k = safe_prefix_len(log["margins"][i], log["scales"][i], prec)
        if k == len(log["margins"][i]):
            assert g == o, (i, g, o)
        else:
            full = False
            assert g[:k] == o[:k], (i, k, g, o)
            # ... and beyond it a valid result of the method under the error bound (A23)
            ok, t = greedy_valid(om, wl.sentence(i), wl.caps[i], g, prec)
            assert ok, ("greedy output not valid under the error bound", i, t, g, o)
        n_cmp += min(k, len(o))
    if full:
        assert st["gen_tokens"] == log["gen_tokens"]
    return n_cmp, st, log


@pytest.mark.parametrize("prec", PRECS)
def test_tiny_free_running_with_pruning(prec):
    wl = tiny_workload(n=8, seed=3)
    n_cmp, st, log = _free_running("tiny", prec, wl, eos_boost=3.0, max_tokens=40, max_sents=3)
    assert n_cmp > (20 if prec == "fp32" else 8)   # FP16: fewer margin-safe positions
    if prec == "fp32":
        assert st["prunes"] == len(log["prunes"])


@pytest.mark.parametrize("prec", PRECS)
def test_prune_maps_bit_exact(prec):
    """Step API with pruning: new_to_old maps equal the oracle's at every decision point."""
    from oracle import translate_fast
    wl = tiny_workload(n=12, seed=5, max_cap=16)
    om = oracle_model("tiny", 3.0)
    log = {}
    translate_fast(om, wl, 4096, 512, prune_ratio=0.25, log=log)
    assert len(log["batches"]) == 1
    order = log["batches"][0]
    srcs = [wl.sentence(i) for i in order]
    caps = wl.caps[order]
    gm = gpu_model("tiny", prec, 3.0, max_tokens=4096, max_sents=64, max_tgt_len=64)
    src, lens = pad_batch(srcs)
    batch = gm.encode(torch.from_numpy(src).cuda(), lens, tgt_cap=caps)
    n = len(order)
    events = []
    t = 0
    while n > 0:
        batch.decode_step(n_live=n)
        n_new, m = batch.prune(ratio=0.25)
        if 0 < n_new < n:
            events.append((t, m.cpu().numpy()[:n_new].tolist()))
        n = n_new
        t += 1
    ref = [(st, keep.tolist()) for (_, st, keep) in log["prunes"]]
    # maps are pinned at every decision point before the first margin-unsafe finish decision
    # of any row of the batch (SURVEY §8(c) prune maps); all of them when every step is safe
    first_unsafe = min(safe_prefix_len(log["margins"][i], log["scales"][i], prec) for i in order)
    pin = lambda ev: [e for e in ev if e[0] < first_unsafe]
    assert pin(events) == pin(ref), (first_unsafe, events, ref)
    if prec == "fp32":
        assert events == ref


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["student-35-1", "student-9-1-tiny"])
def test_35_1_free_running_subset(prec, name):
    """Free-running greedy with pruning vs O-fast: 35-1 (C3) and the CPU-track 9-1-tiny
    (§8(f) f4, d = 256, dh = 32, the CPU batch cap of 64 sentences scaled to 16 here)."""
    wl = newstest_like(40, 32000)
    n_cmp, st, log = _free_running(name, prec, wl, eos_boost=1.0, max_tokens=512, max_sents=16)
    assert n_cmp > 0


def test_translate_host_equals_device_and_steps():
    cfg, _ = weights("student-35-1")
    wl = newstest_like(64, 32000, start=1000)
    gm = gpu_model("student-35-1", "fp16", max_tokens=1024, max_sents=32)
    out_h, st_h = gm.translate(wl.ids, wl.off, caps=wl.caps)
    d_ids = torch.from_numpy(wl.ids).cuda()
    d_out = torch.zeros(wl.n, gm.Tmax, dtype=torch.int32, device="cuda")
    d_len = torch.zeros(wl.n, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()      # non-default stream: CUDA-graph decode steps
    with torch.cuda.stream(side):
        st_d = gm.translate_device(d_ids, wl.off, d_out, d_len, caps=wl.caps)
    torch.cuda.synchronize()
    d_out, d_len = d_out.cpu().numpy(), d_len.cpu().numpy()
    for i in range(wl.n):
        g = d_out[i, :d_len[i]].tolist()
        if g and g[-1] == 3:
            g = g[:-1]
        assert g == out_h[i]
    assert st_h["gen_tokens"] == st_d["gen_tokens"] == int(d_len.sum())
    # deterministic: a second run (graph replay on a side stream) is byte-identical
    with torch.cuda.stream(side):
        out_h2, st2 = gm.translate(wl.ids, wl.off, caps=wl.caps)
    assert out_h2 == out_h
    assert st2["launches"] == st_h["launches"]   # graph replays launch the same kernels
    (flat, offs), _ = gm.translate(wl.ids, wl.off, caps=wl.caps, as_arrays=True)
    assert [flat[offs[i]:offs[i + 1]].tolist() for i in range(wl.n)] == out_h


@pytest.mark.parametrize("prec", PRECS)
def test_beam_tiny_matches_oracle(prec):
    """Batched GPU beam search (K = 4, early stop, pruning, ancestry-indirect KV cache) vs the
    oracle's per-sentence beam search (reading R15)."""
    from oracle import beam_search
    wl = tiny_workload(n=10, seed=11, max_cap=12)
    om = oracle_model("tiny", 3.0)
    ref = [beam_search(om, wl.sentence(i), wl.caps[i], K=4)[0] for i in range(wl.n)]
    gm = gpu_model("tiny", prec, 3.0, max_tokens=256, max_sents=8, max_tgt_len=32, beam=4)
    slp = [oracle_step_logprobs(om, wl.sentence(i)) for i in range(wl.n)]

    def check(out, ref):
        for i, (o, r) in enumerate(zip(out, ref)):
            if prec == "fp32":
                assert o == r, (i, o, r)
            else:   # equal, or a divergence explained by the FP16 error bound
                assert beam_valid(slp[i], wl.caps[i], o, r), (i, o, r)
    for ratio in (0.25, -1.0):
        out, st = gm.translate(wl.ids, wl.off, caps=wl.caps, max_tokens=48, max_sents=4, beam=4,
                               prune_ratio=ratio)
        check(out, ref)
    # K = 1 through the beam machinery is not used by translate (greedy path); K = 2 runs
    out2, _ = gm.translate(wl.ids, wl.off, caps=wl.caps, max_tokens=48, max_sents=4, beam=2)
    ref2 = [beam_search(om, wl.sentence(i), wl.caps[i], K=2)[0] for i in range(wl.n)]
    check(out2, ref2)


@pytest.mark.parametrize("prec", PRECS)
def test_nbest_tiny_matches_oracle(prec):
    """N-best lists (the KD 4-best lists, reading R27): the GPU's N best finished
    hypotheses and their scores vs the oracle's beam_search_nbest; rank 0 equals the 1-best
    translate output."""
    from oracle import beam_search_nbest
    wl = tiny_workload(n=10, seed=11, max_cap=12)
    om = oracle_model("tiny", 3.0)
    gm = gpu_model("tiny", prec, 3.0, max_tokens=256, max_sents=8, max_tgt_len=32, beam=4)
    for K, N in ((4, 4), (4, 2), (3, 3)):
        ref = [beam_search_nbest(om, wl.sentence(i), wl.caps[i], K=K, nbest=N) for i in range(wl.n)]
        hyps, scores, st = gm.translate_nbest(wl.ids, wl.off, N, K, caps=wl.caps, max_tokens=48,
                                              max_sents=4)
        best, _ = gm.translate(wl.ids, wl.off, caps=wl.caps, max_tokens=48, max_sents=4, beam=K)
        assert [h[0] for h in hyps] == best
        for i in range(wl.n):
            if prec == "fp32":
                assert [t for t, _ in ref[i]] == hyps[i], (K, N, i)
                assert all(abs(a - b[1]) <= 1e-4 * max(1.0, abs(b[1])) for a, b in zip(scores[i], ref[i]))
            else:   # rank by rank: equal or within the FP16 bound, GPU score consistent
                slp = oracle_step_logprobs(om, wl.sentence(i))
                for r in range(N):
                    assert beam_valid(slp, wl.caps[i], hyps[i][r], ref[i][r][0], scores[i][r]), (K, N, i, r)
        for sc in scores:   # best first
            assert all(sc[r] >= sc[r + 1] for r in range(len(sc) - 1))


@pytest.mark.parametrize("prec", PRECS)
def test_ensemble_tiny_matches_oracle(prec):
    """Teacher ensemble (reading R26): two tiny members with different
    weights, beam 4 (1-best and 3-best) vs the oracle's beam search over the averaged
    distribution; a one-member ensemble equals the member's own beam search."""
    from synth import generate_weights
    from oracle import OracleModel, beam_search_nbest, ensemble_step_logprobs
    from paper_2109_08008_b200 import Model, Ensemble
    cfg, W1 = weights("tiny", 3.0)
    W2 = generate_weights(cfg, seed=2110, eos_boost=3.0)
    om1, om2 = oracle_model("tiny", 3.0), OracleModel(W2, cfg)
    lim = dict(max_tokens=256, max_sents=8, max_tgt_len=32, beam=4)
    g1 = Model(cfg, W1, precision=prec, **lim)
    g2 = Model(cfg, W2, precision=prec, **lim)
    ens = Ensemble([g1, g2])
    wl = tiny_workload(n=10, seed=12, max_cap=12)
    tol = 1e-4 if prec == "fp32" else 5e-2
    for K, N in ((4, 1), (4, 3)):
        hyps, scores, st = ens.translate(wl.ids, wl.off, beam=K, nbest=N, caps=wl.caps,
                                         max_tokens=48, max_sents=4)
        for i in range(wl.n):
            src = wl.sentence(i)
            slp = ensemble_step_logprobs([om1, om2], src)
            ref = beam_search_nbest(om1, src, wl.caps[i], K=K, nbest=N, step_logprobs=slp)
            if prec == "fp32":
                assert [t for t, _ in ref] == hyps[i], (K, N, i)
                assert all(abs(a - b[1]) <= tol * max(1.0, abs(b[1])) for a, b in zip(scores[i], ref))
            else:
                for r in range(N):
                    assert beam_valid(slp, wl.caps[i], hyps[i][r], ref[r][0], scores[i][r]), (K, N, i, r)
        assert st["sentences"] == wl.n and st["gen_tokens"] > 0
    # graph-replayed ensemble steps (non-default stream) == eager steps, bit for bit
    h_e, s_e, _ = ens.translate(wl.ids, wl.off, beam=4, nbest=3, caps=wl.caps, max_tokens=48,
                                max_sents=4)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for _ in range(2):   # first use of a row bucket runs eagerly, then captured graphs
            h_g, s_g, st_g = ens.translate(wl.ids, wl.off, beam=4, nbest=3, caps=wl.caps,
                                           max_tokens=48, max_sents=4)
    torch.cuda.synchronize()
    assert h_g == h_e and s_g == s_e
    solo = Ensemble([g1])
    hyps, _, _ = solo.translate(wl.ids, wl.off, beam=4, caps=wl.caps, max_tokens=48, max_sents=4)
    best, _ = g1.translate(wl.ids, wl.off, caps=wl.caps, max_tokens=48, max_sents=4, beam=4)
    for i, (h, b) in enumerate(zip(hyps, best)):
        if prec == "fp32":
            assert h[0] == b, i
        elif h[0] != b:   # both valid beam results of the same model under the FP16 bound
            slp = oracle_step_logprobs(om1, wl.sentence(i))
            ref = beam_search_nbest(om1, wl.sentence(i), wl.caps[i], K=4, nbest=1)[0][0]
            assert beam_valid(slp, wl.caps[i], h[0], ref) and beam_valid(slp, wl.caps[i], b, ref), i
    ens.close()
    solo.close()


def test_ensemble_heterogeneous_teachers_subset():
    """Ensemble of two teacher-scale members that differ in depth and DLCL (30-6+DLCL and
    24-6 without DLCL, FP16, beam 4, 2-best) vs the oracle ensemble beam on a subset."""
    from synth import generate_weights
    from oracle import OracleModel, beam_search_nbest, ensemble_step_logprobs
    from paper_2109_08008_b200 import Model, Ensemble
    cfg1, W1 = weights("teacher-30-6")
    cfg2 = PRESETS["teacher-30-6"].replace(enc_layers=24, use_dlcl=False)
    W2 = generate_weights(cfg2, seed=2111)
    om1, om2 = oracle_model("teacher-30-6"), OracleModel(W2, cfg2)
    wl = newstest_like(2, 32000, start=91)
    caps = np.minimum(wl.caps, 6)
    lim = dict(max_tokens=512, max_sents=4, max_tgt_len=16, beam=4)
    ens = Ensemble([Model(cfg1, W1, precision="fp16", **lim), Model(cfg2, W2, precision="fp16", **lim)])
    hyps, scores, _ = ens.translate(wl.ids, wl.off, beam=4, nbest=2, caps=caps)
    for i in range(wl.n):
        src = wl.sentence(i)
        slp = ensemble_step_logprobs([om1, om2], src)
        ref = beam_search_nbest(om1, src, caps[i], K=4, nbest=2, step_logprobs=slp)
        for r in range(2):
            assert beam_valid(slp, caps[i], hyps[i][r], ref[r][0], scores[i][r]), (i, r, hyps[i], ref)
    ens.close()


def test_text_pipeline_end_to_end():
    """§8(f) f3: text lines -> library BPE codec -> GPU greedy translation (tiny, FP32) ->
    codec decode, equal to the oracle pipeline (oracle BPE -> oracle greedy -> oracle
    decode) line for line on margin-safe sentences."""
    from oracle import translate_fast
    from oracle.text import load_merges, load_vocab, bpe_apply, encode_ids, decode_ids, bpe_remove
    from synth import Workload
    from synth.text import synthetic_bpe, synthetic_lines
    from paper_2109_08008_b200 import TextCodec
    m_txt, v_txt, sym = synthetic_bpe(pad_to=1000)
    lines = [ln for ln in synthetic_lines(24, sym, max_words=4) if ln.strip()]
    ranks = load_merges(m_txt)
    tok2id, id2tok = load_vocab(v_txt)
    enc = [encode_ids(bpe_apply(ln, ranks), tok2id) for ln in lines]
    caps = np.full(len(lines), 10, dtype=np.int32)
    om = oracle_model("tiny", 3.0)
    off = np.cumsum([0] + [len(e) for e in enc]).astype(np.int64)
    wl = Workload(np.array(sum(enc, []), dtype=np.int32), off, caps)
    log = {}
    ref_ids = translate_fast(om, wl, max_tokens=256, max_sents=8, log=log)
    ref = [bpe_remove(decode_ids(r, id2tok, 1000)) for r in ref_ids]
    gm = gpu_model("tiny", "fp32", 3.0, max_tokens=256, max_sents=8, max_tgt_len=32)
    codec = TextCodec(v_txt, m_txt)
    got, st = gm.translate_text(codec, lines, caps=caps)
    assert len(got) == len(lines)
    got_ids, _ = gm.translate(wl.ids, wl.off, caps=caps)
    for i in range(len(lines)):
        k = safe_prefix_len(log["margins"][i], log["scales"][i], "fp32")
        if k == len(log["margins"][i]):    # every position margin-safe: the text is pinned
            assert got[i] == ref[i], (i, got[i], ref[i])
        else:
            assert got_ids[i][:k] == ref_ids[i][:k]
            assert greedy_valid(om, wl.sentence(i), caps[i], got_ids[i], "fp32")[0], i
        assert got[i] == bpe_remove(decode_ids(got_ids[i], id2tok, 1000))
    codec.close()


def test_beam_teacher_30_6_subset():
    """C4: teacher-scale 30-6 Transformer-DLCL-RPR, FP16 beam 4 with cached attention."""
    from oracle import beam_search
    wl = newstest_like(3, 32000, start=77)
    caps = np.minimum(wl.caps, 10)
    om = oracle_model("teacher-30-6")
    ref = [beam_search(om, wl.sentence(i), caps[i], K=4)[0] for i in range(wl.n)]
    gm = gpu_model("teacher-30-6", "fp16", max_tokens=512, max_sents=4, max_tgt_len=16, beam=4)
    out, st = gm.translate(wl.ids, wl.off, caps=caps, beam=4)
    for i in range(wl.n):
        assert beam_valid(oracle_step_logprobs(om, wl.sentence(i)), caps[i], out[i], ref[i]), (i, out[i], ref[i])
    assert all(len(o) <= c for o, c in zip(out, caps))


def test_concurrent_workers_identical():
    """n_workers concurrent batch workers (own arena + stream, shared weights) give the
    same outputs as one worker, on host and device paths."""
    wl = newstest_like(300, 32000, start=2000)
    gm = gpu_model("student-6-1", "fp16", max_tokens=1024, max_sents=64, workspaces=3)
    ref, st1 = gm.translate(wl.ids, wl.off, caps=wl.caps)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        for w in (2, 3):
            out, st = gm.translate(wl.ids, wl.off, caps=wl.caps, workers=w)
            assert out == ref
            assert st["gen_tokens"] == st1["gen_tokens"] and st["batches"] == st1["batches"]
        d_ids = torch.from_numpy(wl.ids).cuda()
        d_out = torch.zeros(wl.n, gm.Tmax, dtype=torch.int32, device="cuda")
        d_len = torch.zeros(wl.n, dtype=torch.int32, device="cuda")
        st = gm.translate_device(d_ids, wl.off, d_out, d_len, caps=wl.caps, workers=3)
    torch.cuda.synchronize()
    d_out, d_len = d_out.cpu().numpy(), d_len.cpu().numpy()
    for i in range(wl.n):
        g = d_out[i, :d_len[i]].tolist()
        assert (g[:-1] if g and g[-1] == 3 else g) == ref[i]
    assert st["gen_tokens"] == st1["gen_tokens"]


def test_concurrent_workers_identical_beam():
    """Beam search (30-6 teacher, FP16, beam 4) with 4 concurrent batch workers (the C4
    measurement's setting) gives the same hypotheses and scores as one worker."""
    wl = newstest_like(96, 32000, start=4000)
    caps = np.minimum(wl.caps, 40)
    gm = gpu_model("teacher-30-6", "fp16", max_tokens=1024, max_sents=16, max_tgt_len=40, beam=4,
                   workspaces=4)
    ref, st1 = gm.translate(wl.ids, wl.off, caps=caps, beam=4)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        out, st = gm.translate(wl.ids, wl.off, caps=caps, beam=4, workers=4)
    torch.cuda.synchronize()
    assert out == ref
    assert st["gen_tokens"] == st1["gen_tokens"] and st["batches"] == st1["batches"]


def test_batch_invariance_fp32():
    """Sentence alone == sentence inside a bigger batch (PAPER.md:121 batching is exact)."""
    wl = newstest_like(16, 32000, start=50)
    gm = gpu_model("student-6-1", "fp32", max_tokens=2048, max_sents=64)
    full, _ = gm.translate(wl.ids, wl.off, caps=wl.caps)
    for i in (0, 7, 15):
        one = wl.shard(i, i + 1)
        o, _ = gm.translate(one.ids, one.off, caps=one.caps)
        assert o[0] == full[i]


_LA_SNIPPET = """
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from gpu_common import gpu_model, pad_batch
from synth import newstest_like
wl = newstest_like(48, 32000, start=3000)
src, lens = pad_batch([wl.ids[wl.off[i]:wl.off[i + 1]] for i in range(wl.n)])
out = {{}}
for prec in ("fp32", "fp16"):
    gm = gpu_model("student-35-1", prec, max_tokens=src.size, max_sents=wl.n)
    b = gm.encode(torch.from_numpy(src).cuda(), lens)
    out[prec] = b.encoder_output().cpu().numpy()
np.savez({path!r}, **out)
"""


def test_dlcl_lookahead_bit_identical(tmp_path):
    """The DLCL lookahead (blocks of 2, 3 or 4 boundaries sharing one history read through
    FP32 partials) changes which bytes are read, not the
    arithmetic: the 35-layer encoder output is bit-identical with NMT_NO_DLCL_LA=1 (every
    boundary reads its whole history), FP32 and FP16 modes, for the default block and each
    block size (35 + 1 boundaries: blocks of 3 and 4 end on partial blocks)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    modes = (("la", {}), ("plain", {"NMT_NO_DLCL_LA": "1"}), ("la2", {"NMT_DLCL_LA": "2"}),
             ("la3", {"NMT_DLCL_LA": "3"}), ("la4", {"NMT_DLCL_LA": "4"}))
    for name, env in modes:
        path = str(tmp_path / f"{name}.npz")
        code = _LA_SNIPPET.format(root=root, tests=os.path.join(root, "tests"), path=path)
        e = {k: v for k, v in os.environ.items() if k not in ("NMT_NO_DLCL_LA", "NMT_DLCL_LA")}
        subprocess.run([sys.executable, "-c", code], check=True, env={**e, **env})
        res[name] = np.load(path)
    for name, _ in modes[2:] + modes[:1]:
        for prec in ("fp32", "fp16"):
            assert np.array_equal(res[name][prec], res["plain"][prec]), (name, prec)


def test_decode_gemm_tile_and_split_invariance():
    """The decode GEMM's output tile widens with the launch's row bound and FFN2's split-K
    moves from the cluster kernel to persistent KS = 2 units above 2048 rows (gemm_tc.cu
    decode_config): neither may change a result.  tools/tile_identity.py runs the 35-1 decoder
    projections at 100 / 1000 / 3000 / 8000 rows with tiles 64 / 128 / 256 forced, and the
    library policy against the cluster kernel forced, in child processes (the policy
    switches are read once per process); every output must be bit-identical."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "tile_identity.py"), "100", "1000",
                        "3000", "8000"], capture_output=True, text=True, check=True)
    lines = [l for l in r.stdout.splitlines() if "IDENTICAL" in l or "DIFFER" in l]
    assert len(lines) == 4 * 4 + 4, r.stdout[-2000:]
    assert not [l for l in lines if "DIFFER" in l], r.stdout[-2000:]


def test_step_timing_records():
    """nmt_profile mode 3 + nmt_profile_steps (SURVEY §8(d) ms/decode step): one record per
    graph-replayed decode step, live rows non-increasing within a batch, positive device
    times; the translation is unchanged by the timing; a reset clears the records."""
    wl = newstest_like(96, 32000, start=5000)
    gm = gpu_model("student-35-1", "fp16", max_tokens=2048, max_sents=64)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ref, st0 = gm.translate(wl.ids, wl.off, caps=wl.caps)   # eager first steps, graphs built
        gm.profile(3)
        out, st = gm.translate(wl.ids, wl.off, caps=wl.caps)
        rec = gm.profile_steps()
        gm.profile(0)
    assert out == ref
    assert 0 < len(rec) <= st["decode_steps"]
    assert all(ms > 0 and live >= 1 for _, live, ms in rec)
    for (t0, l0, _), (t1, l1, _) in zip(rec, rec[1:]):
        if t1 == t0 + 1:            # same batch: pruning only shrinks the live set
            assert l1 <= l0
    assert gm.profile_steps() == []


def test_errors():
    from paper_2109_08008_b200 import NmtError
    gm = gpu_model("tiny", "fp16", max_tokens=64, max_sents=4, max_tgt_len=16)
    src = torch.full((5, 4), 5, dtype=torch.int32, device="cuda")
    with pytest.raises(NmtError, match="E_SHAPE"):
        gm.encode(src, [4] * 5)
    with pytest.raises(NmtError, match="E_INPUT"):
        gm.translate(np.array([5, 2000, 3], np.int32), np.array([0, 3]))
