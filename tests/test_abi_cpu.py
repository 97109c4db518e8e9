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
    lim = (ctypes.c_int32 * 4)(4096, 512, 200, 1)
    rc = lib.nmt_load_weights(b"XXXX" + b"\0" * 16, ctypes.c_size_t(20), 0, 1, lim, ctypes.byref(h))
    assert rc == 5  # NMT_E_FORMAT: bad magic is detected before touching the device
    assert b"magic" in lib.nmt_last_error()


def test_ntsd_layout():
    from synth import PRESETS, generate_weights
    from paper_2109_08008_b200 import ntsd
    cfg = PRESETS["tiny"]
    W = generate_weights(cfg)
    blob = ntsd.pack(cfg, W)
    assert blob[:4] == b"NTSD"
    ver, cb = struct.unpack_from("<II", blob, 4)
    assert (ver, cb) == (1, 72)
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
    assert abs(len(ntsd.pack(cfg, W, np.float32)) / len(blob) - 2.0) < 0.05
