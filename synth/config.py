"""Model configurations (hyper-parameters only — no arithmetic of the method).

Shared by the oracle and the CUDA path as *input description*: both sides read
the same numbers, neither side's arithmetic lives here.

Citations (PAPER.md = /root/reference/PAPER.md, line numbers):
  * d=512, 8 heads, 6 decoder layers for teachers, tied embeddings, max relative
    length 8, max position 1024 — PAPER.md:34 (Sec. 2.2 "Training Details").
  * layer-count presets 35-6 / 35-1 / 18-1 / 9-1 — PAPER.md:82-87 (Table 2).
  * teachers 35-6 / 40-6 — PAPER.md:40-43 (Table 1).
  * max source 120 / target 200 — PAPER.md:138 (Sec. 4.4).
  * vocab "32K merge operations using a shared vocabulary" — PAPER.md:31; we
    take V = 32000 (reading R3).
  * FFN width 2048 — not printed; the only value that reproduces the printed
    parameter counts (tests/test_oracle_params.py pins it).
Configs C1..C5 follow BASELINE.json "configs".
"""
from __future__ import annotations

from dataclasses import dataclass, asdict, replace

PAD_ID, UNK_ID, BOS_ID, EOS_ID = 0, 1, 2, 3  # DESIGN.md reading R11


@dataclass(frozen=True)
class ModelConfig:
    enc_layers: int
    dec_layers: int
    d_model: int = 512
    n_heads: int = 8
    d_ffn: int = 2048
    vocab_size: int = 32000
    max_rel_pos: int = 8          # PAPER.md:34 "maximum relative length was 8"
    use_dlcl: bool = True         # Eq. 1-2
    use_rpr: bool = True          # Shaw et al.
    dlcl_ln: bool = True          # test switch for reading A22 (LN inside Eq. 2)
    max_src_len: int = 120
    max_tgt_len: int = 200
    max_pos: int = 1024
    ln_eps: float = 1e-5          # reading R10

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads

    def as_dict(self) -> dict:
        return asdict(self)

    def replace(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


PRESETS = {
    # BASELINE.json configs[0]: 2-layer encoder / 1-layer decoder, d=64, 4 heads, vocab 1000
    "tiny": ModelConfig(enc_layers=2, dec_layers=1, d_model=64, n_heads=4, d_ffn=256,
                        vocab_size=1000, use_dlcl=True, use_rpr=True),
    # configs[1]: student 6-1 base; DLCL off / RPR on (reading R20)
    "student-6-1": ModelConfig(enc_layers=6, dec_layers=1, use_dlcl=False),
    # configs[2] / [4]: 35-1 DLCL+RPR (headline)
    "student-35-1": ModelConfig(enc_layers=35, dec_layers=1),
    # configs[3]: teacher-scale 30-6, beam 4
    "teacher-30-6": ModelConfig(enc_layers=30, dec_layers=6),
    # the paper's other models (parameter-count pins only)
    "student-35-6": ModelConfig(enc_layers=35, dec_layers=6),
    "student-18-1": ModelConfig(enc_layers=18, dec_layers=1),
    "student-9-1": ModelConfig(enc_layers=9, dec_layers=1),
    # §8(f) row f4, the CPU-track model 9-1-tiny: "the same
    # settings as the 9-1 model except that the model size is 256" — reading R30: d = 256,
    # F = 4d = 1024, the 9-1's 8 heads (dh = 32), DLCL + RPR, tied E: 16.4M parameters
    # (the "90%" reduction vs 35-6, and Table 3's 67 MiB as FP32)
    "student-9-1-tiny": ModelConfig(enc_layers=9, dec_layers=1, d_model=256, n_heads=8, d_ffn=1024),
    "teacher-40-6": ModelConfig(enc_layers=40, dec_layers=6),
    # the four ensemble teachers (Table 1), §8(f) row f1
    "ens-35-6": ModelConfig(enc_layers=35, dec_layers=6, use_dlcl=False),
    "ens-35-6-dlcl": ModelConfig(enc_layers=35, dec_layers=6),
    "ens-40-6": ModelConfig(enc_layers=40, dec_layers=6, use_dlcl=False),
    "ens-40-6-dlcl": ModelConfig(enc_layers=40, dec_layers=6),
}
