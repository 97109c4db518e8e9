#!/usr/bin/env python
"""DRAM traffic of the encoder GEMM launches captured by tools/profile.sh (`<tag>_enc_gemm`,
ncu --set full: layer 1's QKV / out-projection / FFN1 / FFN2 launches of the first batch of
chunk 0) next to their algorithmic bytes, written to profiles/<tag>_enc_gemm_traffic.json
for bench.py's roofline `traffic` field.

Usage: python tools/roofline_traffic.py gpurun_out/<tag>_enc_gemm.ncu-rep <tag> [chunk] [max_tokens max_sents]
(the batch budget defaults to bench.py's)"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def first_batch(chunk, max_tokens=131072, max_sents=16384):
    """(B, S) of the first dynamic batch of bench chunk 0 (the paper's rule, DESIGN R17)."""
    from synth import newstest_like
    wl = newstest_like(chunk, 32000, start=0)
    lens = sorted((wl.off[i + 1] - wl.off[i] for i in range(wl.n)), reverse=True)
    S = int(lens[0])
    return min(max_sents, max_tokens // S, wl.n), S


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 1500
    B, S = first_batch(chunk, *[int(x) for x in sys.argv[4:6]]) if len(sys.argv) > 5 else first_batch(chunk)
    M, d, F = B * S, 512, 2048
    # (name, N, K, residual): the launch order of one encoder layer (forward.cu)
    shapes = [("qkv", 3 * d, d, False), ("out", d, d, True), ("ffn1", F, d, False),
              ("ffn2", d, F, True)]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
             "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    def val(r, m):
        i = h.index(m)
        return float(r[i].replace(",", "")) * scale.get(units[i], 1)
    launches = []
    for (name, N, K, res), r in zip(shapes, rows[2:]):
        alg = 2 * (M * K + N * K + M * N + (M * N if res else 0) + N)
        dram = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        launches.append({"gemm": name, "M": M, "N": N, "K": K, "algorithmic_bytes": alg,
                         "dram_bytes": dram, "us": 1e6 * val(r, "gpu__time_duration.sum")})
    n = len(launches)
    res = {"source": f"ncu --set full, {os.path.basename(rep)} (first batch of chunk 0: B={B}, S={S})",
           "launches": launches,
           "dram_bytes_per_launch": sum(x["dram_bytes"] for x in launches) / n,
           "algorithmic_bytes_per_launch": sum(x["algorithmic_bytes"] for x in launches) / n}
    path = os.path.join(ROOT, "profiles", f"{tag}_enc_gemm_traffic.json")
    with open(path, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
