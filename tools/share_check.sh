#!/bin/bash
# Kernel-share cross-check (GPU box): the bench's CUDA-event class shares vs an ncu launch
# list of exactly one bench step of the same command (SHARES must agree; ncu per-launch times
# are serialised and cold-cache).  Usage: bash tools/share_check.sh <tag> [chunk]
tag=${1:-r1g}; chunk=${2:-1500}
out=gpurun_out
B="python bench.py --steps 1 --warmup 0 --chunk $chunk --no-e2e --no-cpu-baseline --no-paper-budget --workers 1"
timeout 600 $B > $out/${tag}_plain.log 2>&1 || exit 1
n=$(python -c "import json;print(json.loads(open('$out/${tag}_plain.log').read().strip().splitlines()[-1])['gpu_launches'])")
echo "timed-step launches: $n"
# the 3 load-time k_fold_ln launches precede the timed step
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 3 -c $n --csv \
  --log-file $out/${tag}_step_launches.csv $B > $out/${tag}_step_ncu.log 2>&1
echo "ncu rc=$?"
