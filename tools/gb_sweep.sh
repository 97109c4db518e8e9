# GEMM tuning sweep (GPU box): encoder-shape GEMM times per kernel configuration
for c in ${CFGS:-default pair256x4 pair256x6}; do for d in ${DBGS:-0}; do echo "== $c dbg=$d"; NMT_GEMM_DBG=$d NMT_GEMM_CFG=$c timeout 300 python tools/gemm_bench.py --tokens 16384 2>&1 | python -c "
import json,sys
t=sys.stdin.read(); i=t.index('{'); d=json.loads(t[i:])
print({k:round(v['us'],1) for k,v in d.items()})
"; done; done
