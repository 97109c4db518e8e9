#!/bin/bash
# Encoder GEMM configuration sweep (GPU box): bash tools/gemm_cfg_sweep.sh [tokens] [cfg ...]
T=${1:-65520}; shift
for c in "${@:-default}"; do
  if [ "$c" = default ]; then python tools/gemm_bench.py --tokens $T; else NMT_GEMM_CFG=$c python tools/gemm_bench.py --tokens $T; fi > /tmp/gb_$c.log 2>&1
  python - $c <<'PY'
import json,sys
t=open(f"/tmp/gb_{sys.argv[1]}.log").read()
try:
    d=json.loads(t[t.index('{'):]); print(sys.argv[1], {k:round(v['us'],1) for k,v in d.items() if k.startswith(('enc','cross'))})
except Exception: print(sys.argv[1], 'ERR', t[-400:])
PY
done
