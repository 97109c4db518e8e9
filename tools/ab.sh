# A/B: bench value with and without an env knob, alternating (GPU box)
knob=${1:-NMT_NO_FOLD}
python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed" | tail -1
for i in 1 2; do
  for v in 0 1; do
    if [ $v = 1 ]; then export $knob=1; else unset $knob; fi
    python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$knob=$v', round(d['value']), round(d['ms_per_step'],1))"
  done
done
