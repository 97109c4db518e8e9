#!/bin/bash
# Workers / chunk sweep at the 131072 / 16384 budget (GPU box)
run() { tag=$1; shift; timeout 600 python bench.py --steps 3 --warmup 3 --no-paper-budget --no-c4 --no-cpu-baseline --no-odef "$@" > /tmp/bs_$tag.log 2>&1
  python - $tag <<'PY'
import json,sys
t=open(f"/tmp/bs_{sys.argv[1]}.log").read()
try:
    d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]); print(sys.argv[1], round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])
except Exception: print(sys.argv[1], 'ERR', t[-300:])
PY
}
run w3_c192 --workers 3
run w4_c192 --workers 4
run w3_c288 --workers 3 --chunk 288000
run w4_c288 --workers 4 --chunk 288000
run w3_c192b --workers 3
run w4_c192b --workers 4
