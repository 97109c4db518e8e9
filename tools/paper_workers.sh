#!/bin/bash
# Paper-budget (4096 / 512) throughput vs concurrent batch workers (GPU box)
for w in "${@:-4 6 8}"; do
  timeout 900 python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline --no-odef --paper-workers $w > /tmp/pw_$w.log 2>&1
  python - $w <<'PY'
import json,sys
t=open(f"/tmp/pw_{sys.argv[1]}.log").read()
try:
    d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]); p=d['paper_budget_tok_s']
    print('paper workers', sys.argv[1], round(p['value']), 'decode_steps', p['decode_steps'], 'main value', round(d['value']))
except Exception: print(sys.argv[1], 'ERR', t[-400:])
PY
done
