#!/bin/bash
# enc_layernorm class A/B helper (GPU box): bench per-class ms, 2 runs
for i in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-paper-budget --no-c4 --no-cpu-baseline --no-odef > /tmp/ln_$i.log 2>&1
  python - $i <<'PY'
import json,sys
t=open(f"/tmp/ln_{sys.argv[1]}.log").read()
try:
    d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]); k=d['kernels']
    print('value', round(d['value']), 'enc_ln', k['enc_layernorm']['ms'], k['enc_layernorm']['frac'], 'dec_ln', k['dec_layernorm']['ms'])
except Exception: print('ERR', t[-500:])
PY
done
