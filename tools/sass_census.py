#!/usr/bin/env python
"""SASS instruction census of libnmt.so (CPU only: cuobjdump -sass): per kernel, the
mnemonics that prove the Blackwell-native paths (B200_PROFILING.md "What proves a
Blackwell-native kernel"): UTCHMMA / UTC*MMA (tcgen05.mma), LDTM / STTM (tcgen05.ld / st),
UTMALDG / UTMASTG / UBLKCP (TMA), UTMAPF (TMA prefetch), HMMA (legacy mma.sync), plus the
instruction count.  Kernels are grouped by demangled base name (template instances summed,
instance count reported).

Usage: python tools/sass_census.py [libnmt.so] [out.json]"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MNEM = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG",
        "UBLKCP", "UTMAPF", "HMMA", "SYNCS", "LDGSTS"]


def base_name(mangled: str) -> str:
    try:
        dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    except Exception:
        dem = mangled
    dem = re.sub(r"\(anonymous namespace\)::", "", dem)
    m = re.match(r"(?:void )?([\w:]+?)(?:<.*)?\(", dem)
    return m.group(1) if m else dem[:60]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2109_08008_b200", "libnmt.so")
    out = sys.argv[2] if len(sys.argv) > 2 else None
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True,
                          text=True).stdout
    per = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            name = base_name(m.group(1))
            cur = per.setdefault(name, {"instances": 0, "instructions": 0,
                                        **{k: 0 for k in MNEM}})
            cur["instances"] += 1
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            cur["instructions"] += 1
            op = m.group(1)
            for k in MNEM:
                if op == k or (k == "UTCHMMA" and op.startswith("UTCHMMA")):
                    cur[k] += 1
                    break
            if op.startswith("UTC") and op.endswith("MMA") and op not in MNEM:
                cur.setdefault(op, 0)
                cur[op] += 1
    res = {"library": os.path.relpath(lib, ROOT), "kernels": per}
    txt = json.dumps(res, indent=1)
    if out:
        with open(out, "w") as f:
            f.write(txt + "\n")
    hdr = f"{'kernel':40s} {'inst':>4s} {'instr':>7s} " + " ".join(f"{k:>7s}" for k in MNEM[:11])
    print(hdr)
    for n, c in per.items():
        print(f"{n[:40]:40s} {c['instances']:4d} {c['instructions']:7d} " +
              " ".join(f"{c[k]:7d}" for k in MNEM[:11]))


if __name__ == "__main__":
    main()
