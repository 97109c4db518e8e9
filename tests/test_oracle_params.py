"""Pin the architecture reading (shapes / tied E / RPR tables / F=2048) to the
parameter counts and FP16 sizes printed in PAPER.md (tests/golden/param_counts.txt)."""
import os

from synth import PRESETS, param_count

GOLD = os.path.join(os.path.dirname(__file__), "golden", "param_counts.txt")


def _golden():
    rows = {}
    for line in open(GOLD):
        line = line.split("#")[0].strip()
        if line:
            name, val, *_ = line.split()
            rows[name] = float(val)
    return rows


def test_param_counts_match_tables():
    g = _golden()
    for name in ("teacher-40-6", "student-35-6", "student-35-1", "student-18-1", "student-9-1"):
        n = param_count(PRESETS[name], include_dlcl=False)
        assert round(n / 1e6) == g[name], (name, n)
    ens = (2 * param_count(PRESETS["student-35-6"], False) + 2 * param_count(PRESETS["teacher-40-6"], False))
    assert round(ens / 1e6) == g["ensemble"]


def test_ensemble_presets_match_table1():
    """The four teacher presets used by the GPU ensemble: each member's
    printed size and the ensemble's 640M (DLCL members counted with their DLCL params)."""
    g = _golden()
    sizes = {n: param_count(PRESETS[n]) for n in ("ens-35-6", "ens-35-6-dlcl", "ens-40-6", "ens-40-6-dlcl")}
    assert round(sizes["ens-35-6"] / 1e6) == round(sizes["ens-35-6-dlcl"] / 1e6) == g["student-35-6"]
    assert round(sizes["ens-40-6"] / 1e6) == round(sizes["ens-40-6-dlcl"] / 1e6) == g["teacher-40-6"]
    assert round(sum(sizes.values()) / 1e6) == g["ensemble"]


def test_dlcl_adds_negligible_params():
    # Table 1 prints the same size with and without DLCL
    for name in ("student-35-6", "teacher-40-6"):
        c = PRESETS[name]
        assert round(param_count(c, True) / 1e6) == round(param_count(c, False) / 1e6)


def test_fp16_file_sizes():
    g = _golden()
    # "291 MiB when stored in 16-bit floats": 152.03M x 2 B = 290.0 MiB
    mib = param_count(PRESETS["student-35-6"], False) * 2 / 2 ** 20
    assert abs(mib - g["fp16_mib:student-35-6"]) <= 1.5
    # Table 3 "MiB" column is MB of FP16 params within ~1% (header / metadata)
    for name in ("student-35-6", "student-35-1", "student-18-1", "student-9-1"):
        mb = param_count(PRESETS[name], False) * 2 / 1e6
        ref = g["fp16_mb:" + name]
        assert 0 <= ref - mb <= 0.012 * ref, (name, mb, ref)


def test_ffn_width_is_2048():
    # F=2048 is the only power-of-two width reproducing 131M for 35-1
    hits = [F for F in (1024, 2048, 4096) if round(param_count(PRESETS["student-35-1"].replace(d_ffn=F), False) / 1e6) == 131]
    assert hits == [2048]


def test_tiny_cpu_model_reading():
    """Reading R30 for 9-1-tiny: 16.4M parameters reproduce the printed ~90%
    reduction vs 35-6 and Table 3's 67 MiB as an FP32 file (within 3%, the other Table 3
    rows are within 1.2% as FP16); the 25M of Table 2 is the contradicting statement."""
    g = _golden()
    n = param_count(PRESETS["student-9-1-tiny"], False)
    red = 1.0 - n / param_count(PRESETS["student-35-6"], False)
    assert abs(red - g["reduction:student-9-1-tiny"]) < 0.015, red
    mb32 = n * 4 / 1e6
    assert 0 <= g["fp32_mib:student-9-1-tiny"] - mb32 <= 0.03 * g["fp32_mib:student-9-1-tiny"], mb32
    # the other widths do not: F = 2048 gives 21.6M (86 MB FP32), 86% reduction
    wide = param_count(PRESETS["student-9-1-tiny"].replace(d_ffn=2048), False)
    assert wide * 4 / 1e6 > 80
