"""-m gpu tests of the fused FP16 decode step (csrc/decode_fused.cu): one persistent kernel
for embedding ... final LN (or fused GEMM segments around the standalone attention kernels
above NMT_FUSE_ROWS live rows) must be bit-identical to the unfused 11-launch step, whose
arithmetic it reproduces (tile shapes, split-K association, epilogue order), for greedy
and beam search, one and six decoder layers; the oracle parity of the fused step itself
follows from this equality and the oracle parity of the unfused step (the fused step is
opt-in: NMT_FUSE_ROWS; measured slower than the graph-replayed unfused step on B200)."""
import os

import numpy as np
import pytest
import torch

from synth import newstest_like
from gpu_common import weights

pytestmark = pytest.mark.gpu


def _model(name, env, **lim):
    from paper_2109_08008_b200 import Model
    cfg, W = weights(name)
    old = {k: os.environ.get(k) for k in ("NMT_NO_FUSE", "NMT_FUSE_ROWS")}
    try:
        for k in old:
            os.environ.pop(k, None)
        os.environ.update(env)
        return Model(cfg, W, precision="fp16", **lim)   # the policy is read at load
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


MODES = {"unfused": {"NMT_NO_FUSE": "1"}, "one_launch": {"NMT_FUSE_ROWS": "100000"},
         "segments": {"NMT_FUSE_ROWS": "0"}, "mixed": {"NMT_FUSE_ROWS": "64"}, "default": {}}


@pytest.mark.parametrize("name,n,lim,beam", [
    ("student-35-1", 600, dict(max_tokens=8192, max_sents=512), 1),
    # the bench budget: live batches up to 8192 rows, 64 row blocks per fused launch
    ("student-35-1", 12000, dict(max_tokens=65536, max_sents=8192, workspaces=4), 1),
    ("student-6-1", 300, dict(max_tokens=2048, max_sents=128), 1),
    ("teacher-30-6", 24, dict(max_tokens=1024, max_sents=16, max_tgt_len=24, beam=4), 4),
])
def test_fused_step_bit_identical(name, n, lim, beam):
    wl = newstest_like(n, 32000, start=5000)
    caps = np.minimum(wl.caps, lim.get("max_tgt_len", 200))
    outs = {}
    side = torch.cuda.Stream()     # graph-replayed steps (first use of a bucket runs eagerly)
    for mode, env in MODES.items():
        m = _model(name, env, **lim)
        wk = lim.get("workspaces", 1)
        with torch.cuda.stream(side):
            o1, st = m.translate(wl.ids, wl.off, caps=caps, beam=beam, workers=wk)
            o2, _ = m.translate(wl.ids, wl.off, caps=caps, beam=beam, workers=wk)
        torch.cuda.synchronize()
        assert o1 == o2, mode
        outs[mode] = (o1, st["gen_tokens"], st["decode_steps"])
        del m
    ref = outs["unfused"]
    for mode, got in outs.items():
        diff = [i for i in range(wl.n) if got[0][i] != ref[0][i]]
        assert not diff, (mode, len(diff), diff[:5])
        assert got[1:] == ref[1:], mode


def test_fused_teacher_forced_logits_identical():
    """Step API with teacher forcing and FP32 logits: fused and unfused steps give the same
    logits bit for bit at every step (35-1, 40 sentences, 14 steps across the clip boundary)."""
    from synth import random_tokens, BOS_ID
    from gpu_common import pad_batch
    wl = newstest_like(40, 32000, start=777)
    srcs = [wl.sentence(i) for i in range(wl.n)]
    src, lens = pad_batch(srcs)
    T = 14
    forced = np.concatenate([np.full((wl.n, 1), BOS_ID), random_tokens(wl.n, T - 1, 32000, seed=8)], 1)
    res = {}
    for mode in ("unfused", "one_launch", "segments"):
        m = _model("student-35-1", MODES[mode], max_tokens=8192, max_sents=64, max_tgt_len=32)
        b = m.encode(torch.from_numpy(src).cuda(), lens)
        lg = []
        for t in range(T):
            r = b.decode_step(prev=torch.from_numpy(forced[:, t].astype(np.int32)).cuda(), logits=True,
                              n_live=wl.n)
            lg.append(r["logits"].cpu().numpy())
            b.prune(ratio=-1.0, want_map=False)
        res[mode] = np.stack(lg)
        del m
    assert np.array_equal(res["unfused"], res["one_launch"])
    assert np.array_equal(res["unfused"], res["segments"])


@pytest.mark.parametrize("name,n,lim", [
    ("tiny", 10, dict(max_tokens=256, max_sents=8, max_tgt_len=32, beam=4)),
    ("teacher-30-6", 16, dict(max_tokens=1024, max_sents=16, max_tgt_len=20, beam=4)),
])
def test_beam_epilogue_matches_logits_path(name, n, lim):
    """FP16 beam: the vocab GEMM's fused epilogue (per 128-column segment LSE partial and
    top-8, merged per row; logits never written) selects the same hypotheses as the FP32-
    logits path (materialised logits + row top-2K); scores agree to FP32 rounding of the
    LSE association."""
    from synth import tiny_workload
    from paper_2109_08008_b200 import Model
    from gpu_common import weights
    if name == "tiny":
        wl = tiny_workload(n=n, seed=11, max_cap=12)
        cfg, W = weights("tiny", 3.0)
    else:
        wl = newstest_like(n, 32000, start=313)
        cfg, W = weights(name)
    caps = np.minimum(wl.caps, lim["max_tgt_len"])
    res = {}
    for mode in ("logits", "epilogue"):
        old = os.environ.pop("NMT_BEAM_EPI", None)
        if mode == "epilogue":
            os.environ["NMT_BEAM_EPI"] = "1"
        try:
            m = Model(cfg, W, precision="fp16", **lim)
        finally:
            os.environ.pop("NMT_BEAM_EPI", None)
            if old is not None:
                os.environ["NMT_BEAM_EPI"] = old
        hyps, scores, _ = m.translate_nbest(wl.ids, wl.off, 2, 4, caps=caps)
        res[mode] = (hyps, scores)
        del m
    (h0, s0), (h1, s1) = res["logits"], res["epilogue"]
    same = sum(a == b for a, b in zip(h0, h1))
    assert same == len(h0), (same, len(h0))
    for a, b in zip(s0, s1):
        for x, y in zip(a, b):
            assert abs(x - y) <= 1e-4 * max(1.0, abs(x)), (x, y)
