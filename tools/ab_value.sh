# A/B of the bench value for an env knob, alternating runs (GPU box): bash tools/ab_value.sh KNOB [VALUE] [ROUNDS]
knob=$1; val=${2:-0}; rounds=${3:-3}
for i in $(seq $rounds); do for v in 0 1; do
  if [ $v = 1 ]; then export $knob=$val; else unset $knob; fi
  python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$knob=' + ('$val' if $v else 'unset'), round(d['value']), round(d['ms_per_step'],1))"
done; done
