#!/bin/bash
# DLCL lookahead block-size A/B on the default bench (GPU box): bash tools/dlcl_ab.sh [blocks ...]
for b in "${@:-2 3 4}"; do
  NMT_DLCL_LA=$b timeout 600 python bench.py --steps 3 --warmup 3 --no-paper-budget --no-c4 --no-cpu-baseline --no-odef > /tmp/dlcl_$b.log 2>&1
  python - $b <<'PY'
import json,sys
t=open(f"/tmp/dlcl_{sys.argv[1]}.log").read()
try:
    d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]); k=d['kernels']['dlcl_combine']
    print('blocks', sys.argv[1], 'value', round(d['value']), 'dlcl_ms', k['ms'], 'frac', k['frac'], 'roof_ms', k['roof_ms'], 'sm_mhz', d['clocks']['sm_mhz'])
except Exception: print(sys.argv[1], 'ERR', t[-500:])
PY
done
