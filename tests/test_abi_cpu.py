"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every
symbol include/nmt.h declares (no compute calls without a GPU); NTSD blob layout."""
import ctypes
import os
import re
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "nmt.h")


def _declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nmt_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2109_08008_b200 import build
    return build.build()


def test_every_declared_symbol_is_exported(libpath):
    lib = ctypes.CDLL(libpath)
    decl = _declared()
    assert len(decl) >= 14
    for name in decl:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for name in decl:
        assert re.search(r"\bT " + name + r"$", out, re.M), name


def test_binding_exports_match_header():
    from paper_2109_08008_b200.nmt import EXPORTS
    assert sorted(EXPORTS) == _declared()


def test_sm100a_cubin(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_last_error_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.nmt_last_error.restype = ctypes.c_char_p
    h = ctypes.c_void_p()
    lim = (ctypes.c_int32 * 5)(4096, 512, 200, 1, 1)
    rc = lib.nmt_load_weights(b"XXXX" + b"\0" * 16, ctypes.c_size_t(20), 0, 1, lim, ctypes.byref(h))
    assert rc == 5  # NMT_E_FORMAT: bad magic is detected before touching the device
    assert b"magic" in lib.nmt_last_error()


def test_ntsd_layout():
    from synth import PRESETS, generate_weights
    from paper_2109_08008_b200 import ntsd
    cfg = PRESETS["tiny"]
    W = generate_weights(cfg)
    blob = ntsd.pack(cfg, W, version=2)
    assert blob[:4] == b"NTSD"
    ver, cb = struct.unpack_from("<II", blob, 4)
    assert (ver, cb) == (2, 72)
    fields = struct.unpack_from("<17if", blob, 12)
    assert fields[:6] == (2, 1, 64, 4, 256, 1000)
    n = struct.unpack_from("<I", blob, 84)[0]
    assert n == len(W)
    # first record is the tied embedding [1000, 64] fp16
    p = 88
    nl = struct.unpack_from("<H", blob, p)[0]
    assert blob[p + 2:p + 2 + nl] == b"emb"
    p += 2 + nl
    dt, nd = struct.unpack_from("<BB", blob, p)
    dims = struct.unpack_from("<2I", blob, p + 2)
    off, nb = struct.unpack_from("<QQ", blob, p + 10)
    assert (dt, nd, dims, nb) == (1, 2, (1000, 64), 1000 * 64 * 2)
    emb = np.frombuffer(blob, dtype=np.float16, count=1000 * 64, offset=off).reshape(1000, 64)
    np.testing.assert_array_equal(emb, W["emb"])
    # FP16 file is half the FP32 one
    assert abs(len(ntsd.pack(cfg, W, np.float32, version=2)) / len(blob) - 2.0) < 0.05


def _spec_blob(cfg, W, dtype=np.float16, flags=None):
    """A checkpoint in the SPEC's v1 byte layout, built here field by field:
    magic, u32 version 1, 8 u32 config (flags bit0 use_dlcl, bit1 shared_emb), u32 count,
    per tensor u16 name_len + name, u8 rank, u32 dims, u8 dtype, inline payload."""
    code = 1 if np.dtype(dtype) == np.float16 else 0
    fl = (int(cfg.use_dlcl) | 2) if flags is None else flags
    b = b"NTSD" + struct.pack("<I", 1)
    b += struct.pack("<8I", cfg.enc_layers, cfg.dec_layers, cfg.d_model, cfg.n_heads, cfg.d_ffn,
                     cfg.vocab_size, cfg.max_rel_pos, fl) + struct.pack("<I", len(W))
    for name, w in W.items():
        a = np.ascontiguousarray(np.asarray(w, dtype=dtype))
        nb = name.encode()
        b += struct.pack("<H", len(nb)) + nb + struct.pack("<B", a.ndim)
        b += b"".join(struct.pack("<I", x) for x in a.shape) + struct.pack("<B", code) + a.tobytes()
    return b


def test_spec_v1_blob_inspects_like_v2():
    from synth import PRESETS, generate_weights
    from paper_2109_08008_b200 import ntsd
    from paper_2109_08008_b200.nmt import ntsd_inspect
    cfg = PRESETS["tiny"]
    W = generate_weights(cfg)
    c1, n1, v1 = ntsd_inspect(_spec_blob(cfg, W))
    c2, n2, v2 = ntsd_inspect(ntsd.pack(cfg, W, version=2))
    assert (v1, v2) == (1, 2) and n1 == n2 == len(W)
    assert abs(c1.pop("ln_eps") - c2.pop("ln_eps")) < 1e-9
    assert c1 == c2
    # the library writer emits exactly the SPEC layout
    assert ntsd.pack(cfg, W) == _spec_blob(cfg, W)
    assert ntsd.pack(cfg, W, np.float32) == _spec_blob(cfg, W, np.float32)
    # FP32 v1 payload is exactly twice the FP16 payload
    assert len(_spec_blob(cfg, W, np.float32)) - len(_spec_blob(cfg, W)) == \
        sum(np.asarray(w).size * 2 for w in W.values())


@pytest.mark.parametrize("mutate,code", [
    ("truncate", 6), ("flags_untied", 9), ("flags_unknown", 5), ("version", 5),
    ("drop_tensor", 6), ("dup_tensor", 6), ("bad_shape", 6)])
def test_ntsd_errors(mutate, code):
    """Format / integrity errors are reported on the host with no device work."""
    from synth import PRESETS, generate_weights
    from paper_2109_08008_b200.nmt import ntsd_inspect, NmtError
    cfg = PRESETS["tiny"]
    W = dict(generate_weights(cfg))
    if mutate == "truncate":
        blob = _spec_blob(cfg, W)[:-3]
    elif mutate == "flags_untied":
        blob = _spec_blob(cfg, W, flags=int(cfg.use_dlcl))
    elif mutate == "flags_unknown":
        blob = _spec_blob(cfg, W, flags=2 | 8)
    elif mutate == "version":
        blob = bytearray(_spec_blob(cfg, W)); blob[4] = 7; blob = bytes(blob)
    elif mutate == "drop_tensor":
        W.pop("dec.final_ln.b"); blob = _spec_blob(cfg, W)
    elif mutate == "dup_tensor":
        blob = _spec_blob(cfg, W)
        blob = blob[:8 + 32] + struct.pack("<I", len(W) + 1) + blob[8 + 36:] + \
            struct.pack("<H", 3) + b"emb" + struct.pack("<BII", 2, 1000, 64) + b"\x01" + \
            np.zeros((1000, 64), np.float16).tobytes()
    else:
        W["emb"] = np.zeros((999, 64)); blob = _spec_blob(cfg, W)
    with pytest.raises(NmtError) as e:
        ntsd_inspect(blob)
    assert e.value.code == code, str(e.value)


def test_ntsd_v2_offset_overflow_is_integrity_error():
    """off + nb must not wrap — an offset near 2^64 with a plausible size is an
    integrity error, not an out-of-bounds read."""
    from synth import PRESETS, generate_weights
    from paper_2109_08008_b200 import ntsd
    from paper_2109_08008_b200.nmt import ntsd_inspect, NmtError
    cfg = PRESETS["tiny"]
    W = generate_weights(cfg)
    blob = bytearray(ntsd.pack(cfg, W, version=2))
    p = 88 + 2 + 3 + 2 + 8          # first record: name "emb", dtype, ndim, 2 dims
    off, nb = struct.unpack_from("<QQ", blob, p)
    struct.pack_into("<Q", blob, p, (1 << 64) - nb + 16)
    with pytest.raises(NmtError) as e:
        ntsd_inspect(bytes(blob))
    assert e.value.code == 6 and "outside the blob" in str(e.value)
    struct.pack_into("<Q", blob, p, off)
    assert ntsd_inspect(bytes(blob))[1] == len(W)
