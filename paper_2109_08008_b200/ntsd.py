"""NTSD weight blob (magic "NTSD", version 1): config block + named FP16/FP32 tensors.

Byte layout (little endian), parsed by csrc/engine.cu:
  "NTSD" | u32 version=1 | u32 config_bytes=72 | nmt_config (17 x i32, 1 x f32)
  | u32 n_tensors | n x { u16 name_len, name, u8 dtype (0 f32, 1 f16), u8 ndim,
  u32 dims[ndim], u64 data_offset (from blob start), u64 nbytes } | 64-aligned data
FP16 parameter files halve the model size.
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


def pack(cfg, weights: dict, dtype=np.float16) -> bytes:
    names = list(weights.keys())
    arrs = [np.ascontiguousarray(np.asarray(weights[n], dtype=dtype)) for n in names]
    code = 1 if np.dtype(dtype) == np.float16 else 0
    head = bytearray(b"NTSD" + struct.pack("<II", 1, 72) + config_block(cfg) + struct.pack("<I", len(names)))
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
