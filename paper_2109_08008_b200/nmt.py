"""Thin ctypes binding over libnmt.so (include/nmt.h): argument marshalling only.

Every step of the translation path runs in the library's sm_100a kernels; PyTorch
provides device buffers and streams.  There is no CPU fallback: if the library is
missing or no CUDA device is present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import ntsd

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnmt.so")

NMT_FP32, NMT_FP16 = 0, 1
STATUS = {0: "OK", 1: "E_ARG", 2: "E_SHAPE", 3: "E_INPUT", 4: "E_STATE", 5: "E_FORMAT",
          6: "E_INTEGRITY", 7: "E_RESOURCE", 8: "E_CUDA", 9: "E_UNSUPPORTED"}

EXPORTS = ["nmt_load_weights", "nmt_get_config", "nmt_free_model", "nmt_encode",
           "nmt_batch_encoder_output", "nmt_decode_step", "nmt_prune_batch", "nmt_batch_live",
           "nmt_batch_results", "nmt_translate", "nmt_translate_device", "nmt_last_error",
           "nmt_dev_gemm", "nmt_dev_gemm_argmax", "nmt_profile", "nmt_dev_gemm_decode",
           "nmt_translate_nbest", "nmt_ensemble_create", "nmt_ensemble_free",
           "nmt_translate_ensemble", "nmt_text_load", "nmt_text_free", "nmt_text_vocab_size",
           "nmt_text_encode", "nmt_text_decode", "nmt_dev_attn_encoder",
           "nmt_profile_steps", "nmt_batch_free", "nmt_ntsd_inspect", "nmt_debug_fused_trace", "nmt_debug_attn_trace", "nmt_debug_gemm_trace"]


class ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double),
                ("flops", C.c_double), ("bytes", C.c_double)]


class StepRec(C.Structure):
    _fields_ = [("t", C.c_int32), ("n_live", C.c_int32), ("ms", C.c_float)]


class NmtError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Limits(C.Structure):
    _fields_ = [("max_tokens", C.c_int32), ("max_sents", C.c_int32), ("max_tgt_len", C.c_int32),
                ("beam", C.c_int32), ("n_workspaces", C.c_int32)]


class Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "enc_layers", "dec_layers", "d_model", "n_heads", "d_ffn", "vocab_size", "max_rel_pos",
        "use_dlcl", "use_rpr", "dlcl_ln", "max_src_len", "max_tgt_len", "max_pos", "pad_id",
        "unk_id", "bos_id", "eos_id")] + [("ln_eps", C.c_float)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class StepOut(C.Structure):
    _fields_ = [("d_next", C.c_void_p), ("d_parent", C.c_void_p), ("d_score", C.c_void_p),
                ("d_done", C.c_void_p), ("d_logits", C.c_void_p)]


class TranslateOpts(C.Structure):
    _fields_ = [("max_tokens", C.c_int32), ("max_sents", C.c_int32), ("prune_every", C.c_int32),
                ("prune_ratio", C.c_float), ("sync_every", C.c_int32), ("h_tgt_cap", C.c_void_p),
                ("n_workers", C.c_int32), ("beam", C.c_int32), ("nbest", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("sentences", "src_tokens", "gen_tokens", "out_tokens",
                                         "decode_steps", "prunes", "batches", "launches",
                                         "truncated", "arena_system_allocs")] + \
               [("ms_total", C.c_double), ("ms_encode", C.c_double), ("ms_decode", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_lib = None


def lib():
    """Load libnmt.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2109_08008_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.nmt_last_error.restype = C.c_char_p
        for n in EXPORTS:
            getattr(L, n)
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise NmtError(code, lib().nmt_last_error().decode())


def ntsd_inspect(blob: bytes):
    """Host-only NTSD parse + validation (C-ABI nmt_ntsd_inspect; no device needed).
    Returns (config dict, tensor count, version)."""
    cfg = Config()
    nt = C.c_int64()
    ver = C.c_int32()
    _check(lib().nmt_ntsd_inspect(blob, C.c_size_t(len(blob)), C.byref(cfg), C.byref(nt), C.byref(ver)))
    return cfg.as_dict(), nt.value, ver.value


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Model:
    """A loaded model (weights + arena) on one CUDA device."""

    def __init__(self, cfg, weights: dict, precision: str = "fp16", max_tokens: int = 4096,
                 max_sents: int = 512, max_tgt_len: int | None = None, device: int = 0,
                 beam: int = 1, workspaces: int = 1, ntsd_version=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libnmt needs a CUDA device (no CPU fallback)")
        self.cfg = cfg
        self.prec = NMT_FP16 if precision == "fp16" else NMT_FP32
        self.device = device
        self.V = cfg.vocab_size
        self.Tmax = max_tgt_len or cfg.max_tgt_len
        blob = ntsd.pack(cfg, weights, version=ntsd_version)
        lim = Limits(max_tokens, max_sents, self.Tmax, beam, workspaces)
        h = C.c_void_p()
        torch.cuda.set_device(device)
        _check(lib().nmt_load_weights(blob, C.c_size_t(len(blob)), device, self.prec, C.byref(lim),
                                      C.byref(h)))
        self.h = h
        self.limits = lim

    def __del__(self):
        if getattr(self, "h", None):
            lib().nmt_free_model(self.h)
            self.h = None

    def profile(self, mode: int = -1):
        """mode 1 enable, 2 reset+enable, 0 reset+disable, -1 read.  Returns
        {class: {launches, ms, flops, bytes}} read before any reset."""
        buf = (ProfEntry * 16)()
        n = C.c_int32()
        _check(lib().nmt_profile(self.h, mode, buf, 16, C.byref(n)))
        return {buf[i].name.decode(): {"launches": buf[i].launches, "ms": buf[i].ms,
                                       "flops": buf[i].flops, "bytes": buf[i].bytes}
                for i in range(n.value)}

    def profile_steps(self):
        """Decode steps recorded while profiling: list of (t, live rows, device ms)."""
        n = C.c_int32()
        _check(lib().nmt_profile_steps(self.h, None, 0, C.byref(n)))
        buf = (StepRec * max(1, n.value))()
        _check(lib().nmt_profile_steps(self.h, buf, n.value, C.byref(n)))
        return [(buf[i].t, buf[i].n_live, buf[i].ms) for i in range(n.value)]

    # ---------------------------------------------------------------- step API
    def encode(self, src, src_len, tgt_cap=None, beam=1, stream=None):
        """src: int32 CUDA tensor [B][S] (PAD-filled); src_len / tgt_cap: host ints."""
        B, S = src.shape
        ln = np.ascontiguousarray(src_len, dtype=np.int32)
        cp = None if tgt_cap is None else np.ascontiguousarray(tgt_cap, dtype=np.int32)
        b = C.c_void_p()
        _check(lib().nmt_encode(self.h, _ptr(src), ln.ctypes.data_as(C.c_void_p),
                                None if cp is None else cp.ctypes.data_as(C.c_void_p), B, S, beam,
                                _stream(stream), C.byref(b)))
        return Batch(self, b, B, S)

    def translate(self, ids, off, caps=None, max_tokens=None, max_sents=None, prune_every=1,
                  prune_ratio=0.25, sync_every=4, workers=1, beam=1, stream=None, as_arrays=False):
        """Host-buffer translation (C-ABI nmt_translate). Returns (outputs, stats dict);
        outputs = one token list per sentence, or with as_arrays=True the library's flat
        (ids int32 [total], offsets int64 [n+1]) buffers as returned (no per-sentence lists)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        off = np.ascontiguousarray(off, dtype=np.int64)
        n = len(off) - 1
        capa = None if caps is None else np.ascontiguousarray(caps, dtype=np.int32)
        o = TranslateOpts(max_tokens or self.limits.max_tokens, max_sents or self.limits.max_sents,
                          prune_every, prune_ratio, sync_every,
                          None if capa is None else capa.ctypes.data, workers, beam)
        out_cap = n * self.Tmax
        out = np.empty(max(out_cap, 1), dtype=np.int32)
        out_off = np.empty(n + 1, dtype=np.int64)
        st = Stats()
        _check(lib().nmt_translate(self.h, ids.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p),
                                   C.c_int64(n), C.byref(o), out.ctypes.data_as(C.c_void_p),
                                   C.c_int64(out_cap), out_off.ctypes.data_as(C.c_void_p), C.byref(st),
                                   _stream(stream)))
        if as_arrays:
            return (out[:out_off[n]], out_off), st.as_dict()
        outs = [out[out_off[i]:out_off[i + 1]].tolist() for i in range(n)]
        return outs, st.as_dict()

    def translate_text(self, codec, lines, caps=None, threads=4, **kw):
        """File-to-file path (§8(f) f3): lines -> BPE ids (library codec) -> nmt_translate
        -> ids -> lines with the separators removed."""
        ids, off = codec.encode(lines, threads=threads)
        outs, st = self.translate(ids, off, caps=caps, **kw)
        oo = np.cumsum([0] + [len(o) for o in outs]).astype(np.int64)
        flat = np.array([t for o in outs for t in o], dtype=np.int32)
        return codec.decode(flat, oo), st

    def translate_nbest(self, ids, off, nbest, beam, caps=None, max_tokens=None, max_sents=None,
                        prune_every=1, prune_ratio=0.25, sync_every=4, workers=1, stream=None):
        """N-best beam translation (C-ABI nmt_translate_nbest).  Returns
        ([[tokens of rank 0..N-1] per sentence], [[scores]], stats dict)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        off = np.ascontiguousarray(off, dtype=np.int64)
        n = len(off) - 1
        capa = None if caps is None else np.ascontiguousarray(caps, dtype=np.int32)
        o = TranslateOpts(max_tokens or self.limits.max_tokens, max_sents or self.limits.max_sents,
                          prune_every, prune_ratio, sync_every,
                          None if capa is None else capa.ctypes.data, workers, beam, nbest)
        out_cap = n * nbest * self.Tmax
        out = np.empty(max(out_cap, 1), dtype=np.int32)
        out_off = np.empty(n * nbest + 1, dtype=np.int64)
        score = np.empty(max(n * nbest, 1), dtype=np.float32)
        st = Stats()
        _check(lib().nmt_translate_nbest(self.h, ids.ctypes.data_as(C.c_void_p),
                                         off.ctypes.data_as(C.c_void_p), C.c_int64(n), C.byref(o),
                                         out.ctypes.data_as(C.c_void_p), C.c_int64(out_cap),
                                         out_off.ctypes.data_as(C.c_void_p),
                                         score.ctypes.data_as(C.c_void_p), C.byref(st),
                                         _stream(stream)))
        hyps = [[out[out_off[i * nbest + r]:out_off[i * nbest + r + 1]].tolist() for r in range(nbest)]
                for i in range(n)]
        scores = [[float(score[i * nbest + r]) for r in range(nbest)] for i in range(n)]
        return hyps, scores, st.as_dict()

    def translate_device(self, d_ids, off, d_out, d_out_len, caps=None, max_tokens=None,
                         max_sents=None, prune_every=1, prune_ratio=0.25, sync_every=4, workers=1,
                         beam=1,
                         stream=None):
        """Device-resident translation (C-ABI nmt_translate_device); d_out [n][stride]."""
        off = np.ascontiguousarray(off, dtype=np.int64)
        n = len(off) - 1
        capa = None if caps is None else np.ascontiguousarray(caps, dtype=np.int32)
        o = TranslateOpts(max_tokens or self.limits.max_tokens, max_sents or self.limits.max_sents,
                          prune_every, prune_ratio, sync_every,
                          None if capa is None else capa.ctypes.data, workers, beam)
        st = Stats()
        _check(lib().nmt_translate_device(self.h, _ptr(d_ids), off.ctypes.data_as(C.c_void_p),
                                          C.c_int64(n), C.byref(o), _ptr(d_out),
                                          C.c_int32(d_out.shape[1]), _ptr(d_out_len), C.byref(st),
                                          _stream(stream)))
        self._keep = capa
        return st.as_dict()


class Batch:
    def __init__(self, model, h, B, S):
        self.model, self.h, self.B, self.S = model, h, B, S
        self.step = 0

    def encoder_output(self, stream=None):
        import torch
        out = torch.empty(self.B, self.S, self.model.cfg.d_model, dtype=torch.float32, device="cuda")
        _check(lib().nmt_batch_encoder_output(self.h, _ptr(out), _stream(stream)))
        return out

    def decode_step(self, prev=None, logits=False, n_live=None, stream=None):
        """One step; returns dict of CUDA tensors next / parent / score / done (/ logits) for
        the live rows (score: beam only)."""
        import torch
        rows = n_live if n_live is not None else self.live(stream)
        nxt = torch.empty(max(rows, 1), dtype=torch.int32, device="cuda")
        par = torch.empty(max(rows, 1), dtype=torch.int32, device="cuda")
        sc = torch.full((max(rows, 1),), float("nan"), dtype=torch.float32, device="cuda")
        done = torch.empty(max(rows, 1), dtype=torch.uint8, device="cuda")
        lg = torch.empty(max(rows, 1), self.model.V, dtype=torch.float32, device="cuda") if logits else None
        so = StepOut(nxt.data_ptr(), par.data_ptr(), sc.data_ptr(), done.data_ptr(),
                     0 if lg is None else lg.data_ptr())
        _check(lib().nmt_decode_step(self.model.h, self.h, _ptr(prev), self.step, C.byref(so),
                                     _stream(stream)))
        r = {"next": nxt[:rows], "parent": par[:rows], "score": sc[:rows], "done": done[:rows]}
        if lg is not None:
            r["logits"] = lg[:rows]
        return r

    def prune(self, ratio=0.25, want_map=True, keep=None, stream=None):
        """nmt_prune_batch: ratio rule, or the caller's keep mask (uint8 CUDA tensor [n_live])."""
        import torch
        rows = self.live(stream)
        m = torch.empty(max(rows, 1), dtype=torch.int32, device="cuda") if want_map else None
        n = C.c_int32()
        _check(lib().nmt_prune_batch(self.model.h, self.h, C.c_float(ratio), _ptr(keep), _ptr(m),
                                     C.byref(n), _stream(stream)))
        self.step += 1
        return n.value, (m[:rows] if m is not None else None)

    def free(self):
        """nmt_batch_free: the arena is released for the next encode; the handle is dead."""
        if self.h:
            lib().nmt_batch_free(self.h)
            self.h = None

    def live(self, stream=None):
        n = C.c_int32()
        _check(lib().nmt_batch_live(self.h, C.byref(n), _stream(stream)))
        return n.value

    def results(self, stream=None):
        ids = np.empty((self.B, self.model.Tmax), dtype=np.int32)
        ln = np.empty(self.B, dtype=np.int32)
        _check(lib().nmt_batch_results(self.h, ids.ctypes.data_as(C.c_void_p), ln.ctypes.data_as(C.c_void_p),
                                       _stream(stream)))
        return ids, ln


def dev_gemm(A, B, bias=None, R=None, relu=False, out=None, stream=None):
    """C = A B^T (+bias) (+R) (relu) through the library GEMM (fp16: tcgen05; fp32: SIMT)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    prec = NMT_FP16 if A.dtype == torch.float16 else NMT_FP32
    C_ = out if out is not None else torch.empty(M, N, dtype=A.dtype, device=A.device)
    _check(lib().nmt_dev_gemm(prec, M, N, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(bias),
                              _ptr(R), 0 if R is None else R.stride(0), _ptr(C_), C_.stride(0),
                              int(relu), _stream(stream)))
    return C_


def dev_gemm_decode(A, B, bias=None, R=None, relu=False, out=None, stream=None):
    """FP16 GEMM in the decode-step configuration (64-wide tiles, deterministic split-K)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    C_ = out if out is not None else torch.empty(M, N, dtype=A.dtype, device=A.device)
    _check(lib().nmt_dev_gemm_decode(M, N, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0), _ptr(bias),
                                     _ptr(R), 0 if R is None else R.stride(0), _ptr(C_), C_.stride(0),
                                     int(relu), _stream(stream)))
    return C_


def dev_gemm_argmax(A, B, logits=False, stream=None):
    import torch
    M, K = A.shape
    N = B.shape[0]
    prec = NMT_FP16 if A.dtype == torch.float16 else NMT_FP32
    nxt = torch.empty(M, dtype=torch.int32, device=A.device)
    lg = torch.empty(M, N, dtype=torch.float32, device=A.device) if logits else None
    _check(lib().nmt_dev_gemm_argmax(prec, M, N, K, _ptr(A), A.stride(0), _ptr(B), B.stride(0),
                                     _ptr(nxt), _ptr(lg), _stream(stream)))
    return (nxt, lg) if logits else nxt


def dev_attn_encoder(qkv, lens, relk, relv, B, S, H, kclip, use_rpr=True, stream=None):
    """Encoder RPR self-attention alone (C-ABI nmt_dev_attn_encoder): qkv [B*S][3d] CUDA
    tensor (fp16 / fp32), lens int32 CUDA [B], relk / relv [2k+1][dh]; returns out [B*S][d]."""
    import torch
    d = qkv.shape[1] // 3
    prec = NMT_FP16 if qkv.dtype == torch.float16 else NMT_FP32
    out = torch.empty(B * S, d, dtype=qkv.dtype, device=qkv.device)
    _check(lib().nmt_dev_attn_encoder(prec, B, S, d, H, kclip, int(use_rpr), _ptr(qkv), _ptr(lens),
                                      _ptr(relk), _ptr(relv), _ptr(out), _stream(stream)))
    return out


class Ensemble:
    """Teacher ensemble (C-ABI nmt_ensemble_*): member Models with one
    vocabulary decode together; per beam step their distributions are averaged (R26)."""

    def __init__(self, models):
        self.models = list(models)   # the members must outlive the ensemble
        arr = (C.c_void_p * len(self.models))(*[m.h for m in self.models])
        h = C.c_void_p()
        _check(lib().nmt_ensemble_create(arr, C.c_int32(len(self.models)), C.byref(h)))
        self.h = h
        self.Tmax = self.models[0].Tmax
        self.limits = self.models[0].limits

    def close(self):
        if getattr(self, "h", None):
            lib().nmt_ensemble_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def translate(self, ids, off, beam, nbest=1, caps=None, max_tokens=None, max_sents=None,
                  prune_every=1, prune_ratio=0.25, sync_every=4, stream=None):
        """Returns ([[tokens of rank 0..N-1]] per sentence, [[scores]], stats), N = nbest."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        off = np.ascontiguousarray(off, dtype=np.int64)
        n = len(off) - 1
        N = max(1, nbest)
        capa = None if caps is None else np.ascontiguousarray(caps, dtype=np.int32)
        o = TranslateOpts(max_tokens or self.limits.max_tokens, max_sents or self.limits.max_sents,
                          prune_every, prune_ratio, sync_every,
                          None if capa is None else capa.ctypes.data, 1, beam, nbest)
        out_cap = n * N * self.Tmax
        out = np.empty(max(out_cap, 1), dtype=np.int32)
        out_off = np.empty(n * N + 1, dtype=np.int64)
        score = np.empty(max(n * N, 1), dtype=np.float32)
        st = Stats()
        _check(lib().nmt_translate_ensemble(self.h, ids.ctypes.data_as(C.c_void_p),
                                            off.ctypes.data_as(C.c_void_p), C.c_int64(n),
                                            C.byref(o), out.ctypes.data_as(C.c_void_p),
                                            C.c_int64(out_cap), out_off.ctypes.data_as(C.c_void_p),
                                            score.ctypes.data_as(C.c_void_p), C.byref(st),
                                            _stream(stream)))
        hyps = [[out[out_off[i * N + r]:out_off[i * N + r + 1]].tolist() for r in range(N)]
                for i in range(n)]
        scores = [[float(score[i * N + r]) for r in range(N)] for i in range(n)]
        return hyps, scores, st.as_dict()


class TextCodec:
    """Host-side text pipeline (C-ABI nmt_text_*): fastBPE-style subword
    codec + shared vocabulary.  encode(lines) -> (ids, off); decode(ids, off) -> lines."""

    def __init__(self, vocab_text: str, merges_text: str):
        v = vocab_text.encode("utf-8")
        m = merges_text.encode("utf-8")
        h = C.c_void_p()
        _check(lib().nmt_text_load(v, C.c_int64(len(v)), m, C.c_int64(len(m)), C.byref(h)))
        self.h = h

    @property
    def vocab_size(self):
        L = lib()
        L.nmt_text_vocab_size.restype = C.c_int32
        return int(L.nmt_text_vocab_size(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().nmt_text_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def encode(self, lines, threads=1):
        text = "\n".join(lines).encode("utf-8")
        n = len(lines)
        cap = len(text) + 2 * n + 16          # at most one id per byte + EOS per line
        ids = np.empty(cap, dtype=np.int32)
        off = np.empty(n + 2, dtype=np.int64)
        nl = C.c_int64()
        _check(lib().nmt_text_encode(self.h, text, C.c_int64(len(text)), C.c_int32(threads),
                                     ids.ctypes.data_as(C.c_void_p), C.c_int64(cap),
                                     off.ctypes.data_as(C.c_void_p), C.c_int64(n + 1), C.byref(nl)))
        k = int(nl.value)
        # an empty trailing line is not a line
        return ids[: off[k]].copy(), off[: k + 1].copy()

    def decode(self, ids, off):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        off = np.ascontiguousarray(off, dtype=np.int64)
        n = len(off) - 1
        cap = 64 * (len(ids) + 1) + n + 16
        buf = C.create_string_buffer(cap)
        ol = C.c_int64()
        _check(lib().nmt_text_decode(self.h, ids.ctypes.data_as(C.c_void_p),
                                     off.ctypes.data_as(C.c_void_p), C.c_int64(n), buf,
                                     C.c_int64(cap), C.byref(ol)))
        return buf.raw[: ol.value].decode("utf-8").split("\n")[:n]

