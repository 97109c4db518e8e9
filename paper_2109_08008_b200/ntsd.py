"""NTSD weight blob writer (the reader is csrc/engine.cu parse_blob; include/nmt.h).

Two little-endian layouts, both magic "NTSD" (FP16 halves the model):
  v1 — the SPEC checkpoint layout: u32 version=1 | 8 x u32 config (enc_layers, dec_layers,
       d_model, n_heads, d_ffn, vocab_size, max_rel_pos (0 = no RPR), flags: bit0 use_dlcl,
       bit1 shared_emb) | u32 n_tensors | n x { u16 name_len, name, u8 rank, u32 dims[rank],
       u8 dtype (0 f32, 1 f16), payload inline }.  The remaining fields take the DESIGN.md
       readings (dlcl_ln on, max lengths 120 / 200, 1024 positions, ids 0..3, eps 1e-5).
  v2 — this build's extended layout for configs v1 cannot express (e.g. the dlcl_ln test
       switch): u32 version=2 | u32 72 | nmt_config (17 x i32, 1 x f32) | u32 n_tensors |
       n x { u16 name_len, name, u8 dtype, u8 ndim, u32 dims[ndim], u64 data_offset, u64 nbytes }
       | 64-aligned data.
pack() writes v1 whenever the config is expressible in it.
"""
from __future__ import annotations

import struct

import numpy as np

_CFG_FMT = "<17if"
PAD_ID, UNK_ID, BOS_ID, EOS_ID = 0, 1, 2, 3  # reading R11


def config_block(cfg) -> bytes:
    return struct.pack(_CFG_FMT, cfg.enc_layers, cfg.dec_layers, cfg.d_model, cfg.n_heads, cfg.d_ffn,
                       cfg.vocab_size, cfg.max_rel_pos, int(cfg.use_dlcl), int(cfg.use_rpr),
                       int(cfg.dlcl_ln), cfg.max_src_len, cfg.max_tgt_len, cfg.max_pos, PAD_ID, UNK_ID,
                       BOS_ID, EOS_ID, float(cfg.ln_eps))


def v1_expressible(cfg) -> bool:
    return (bool(cfg.dlcl_ln) and cfg.max_src_len == 120 and cfg.max_tgt_len == 200
            and cfg.max_pos == 1024 and abs(cfg.ln_eps - 1e-5) < 1e-12)


def pack_v1(cfg, weights: dict, dtype=np.float16) -> bytes:
    code = 1 if np.dtype(dtype) == np.float16 else 0
    flags = (1 if cfg.use_dlcl else 0) | 2
    out = bytearray(b"NTSD" + struct.pack("<I", 1))
    out += struct.pack("<8I", cfg.enc_layers, cfg.dec_layers, cfg.d_model, cfg.n_heads, cfg.d_ffn,
                       cfg.vocab_size, cfg.max_rel_pos if cfg.use_rpr else 0, flags)
    out += struct.pack("<I", len(weights))
    for n, w in weights.items():
        a = np.ascontiguousarray(np.asarray(w, dtype=dtype))
        nb = n.encode()
        out += struct.pack("<H", len(nb)) + nb + struct.pack("<B", a.ndim)
        out += struct.pack("<%dI" % a.ndim, *a.shape) + struct.pack("<B", code) + a.tobytes()
    return bytes(out)


def pack_v2(cfg, weights: dict, dtype=np.float16) -> bytes:
    names = list(weights.keys())
    arrs = [np.ascontiguousarray(np.asarray(weights[n], dtype=dtype)) for n in names]
    code = 1 if np.dtype(dtype) == np.float16 else 0
    head = bytearray(b"NTSD" + struct.pack("<II", 2, 72) + config_block(cfg) + struct.pack("<I", len(names)))
    recs = []
    for n, a in zip(names, arrs):
        nb = n.encode()
        recs.append(struct.pack("<H", len(nb)) + nb + struct.pack("<BB", code, a.ndim) +
                    struct.pack("<%dI" % a.ndim, *a.shape))
    hdr_len = len(head) + sum(len(r) + 16 for r in recs)
    off = (hdr_len + 63) & ~63
    data = bytearray()
    offsets = []
    for a in arrs:
        offsets.append(off + len(data))
        data += a.tobytes()
        pad = (-len(data)) % 64
        data += b"\0" * pad
    for r, a, o in zip(recs, arrs, offsets):
        head += r + struct.pack("<QQ", o, a.nbytes)
    head += b"\0" * (off - len(head))
    return bytes(head + data)


def pack(cfg, weights: dict, dtype=np.float16, version=None) -> bytes:
    if version is None:
        version = 1 if v1_expressible(cfg) else 2
    return pack_v1(cfg, weights, dtype) if version == 1 else pack_v2(cfg, weights, dtype)
