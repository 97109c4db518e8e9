#!/usr/bin/env python
"""Compare the bench's per-class kernel shares (CUDA events, `kernels` in the JSON line)
with an ncu launch list of exactly one bench step of the same command (tools/share_check.sh).
Launches are classified by kernel name and, for the names both phases use, by position: a
launch between a decoder embedding (k_embed_dec_ln_vec) and the step's finish/prune kernel
belongs to the decode step (the vocab GEMM is the 256-wide GEMM there).
Usage: python tools/share_compare.py <plain.log> <step_launches.csv>"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import load  # noqa: E402


def classify(rows):
    out = []
    in_dec = False
    for name, us, _ in rows:
        n = name.split("::")[-1]
        if "k_embed_dec_ln" in n:
            in_dec = True
            out.append(("embed", us))
            continue
        if "k_finish_prune" in n or "k_beam_select" in n or "k_prune" in n:
            out.append(("bookkeeping", us))
            in_dec = False
            continue
        if n.startswith("k_embed"):
            cls = "embed"
        elif "k_dlcl" in n:
            cls = "dlcl_combine"
        elif "k_attn_enc" in n:
            cls = "enc_rpr_attn"
        elif "k_attn_dec_self" in n:
            cls = "dec_self_attn"
        elif "k_attn_cross" in n:
            cls = "dec_cross_attn"
        elif "k_layernorm" in n:
            cls = "dec_layernorm" if in_dec else "enc_layernorm"
        elif "k_gemm_tc" in n:
            if in_dec:
                cls = "vocab_argmax" if "<256" in n else "dec_gemm"
            else:
                cls = "enc_gemm"
        else:
            cls = "other (" + n.split("<")[0] + ")"
        out.append((cls, us))
    return out


def main():
    line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    ev = {k: v["ms"] for k, v in line["kernels"].items()}
    tot_ev = sum(ev.values())
    nc = {}
    for cls, us in classify(load(sys.argv[2])):
        nc[cls] = nc.get(cls, 0.0) + us
    tot_nc = sum(v for k, v in nc.items() if not k.startswith("other"))
    print(f"{'class':20s} {'bench ms':>10s} {'share':>7s} {'ncu ms':>10s} {'share':>7s}")
    for k in sorted(set(ev) | set(nc), key=lambda c: -ev.get(c, 0.0)):
        a, b = ev.get(k, 0.0), nc.get(k, 0.0)
        sa = f"{a / tot_ev:7.3f}" if k in ev else "      -"
        sb = f"{b / tot_nc:7.3f}" if not k.startswith("other") and k in nc else "      -"
        print(f"{k:20s} {a:10.2f} {sa} {b / 1e3:10.2f} {sb}")
    print(f"{'total':20s} {tot_ev:10.2f} {'':7s} {tot_nc / 1e3:10.2f}")


if __name__ == "__main__":
    main()
