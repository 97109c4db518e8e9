#!/bin/bash
# Batch-budget / worker sweep of the default bench (GPU box): bash tools/budget_sweep.sh
run() { tag=$1; shift; timeout 500 python bench.py --steps 3 --warmup 3 --no-paper-budget --no-c4 --no-cpu-baseline --no-odef "$@" > gpurun_out/sweep_$tag.log 2>&1;
  python - $tag <<'PY'
import json,sys
t=open(f"gpurun_out/sweep_{sys.argv[1]}.log").read()
try:
    d=json.loads([l for l in t.splitlines() if l.startswith('{')][-1]); print(sys.argv[1], round(d['value']), round(d['e2e']['value']), d['ms_per_step'], d['clocks']['sm_mhz'])
except Exception as e: print(sys.argv[1], 'ERR', t[-300:])
PY
}
run ${SWEEP_BASE:-base} 
run t131k_w4_c192 --max-tokens 131072 --max-sents 16384 --workers 4 --chunk 192000
run t131k_w3_c288 --max-tokens 131072 --max-sents 16384 --workers 3 --chunk 288000
run t196k_w3_c192 --max-tokens 196608 --max-sents 24576 --workers 3 --chunk 192000
run t196k_w2_c192 --max-tokens 196608 --max-sents 24576 --workers 2 --chunk 192000
run t131k_w3_c192 --max-tokens 131072 --max-sents 16384 --workers 3 --chunk 192000
