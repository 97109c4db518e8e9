# A/B on the per-class profile (workers=1 serial kernel times, stabler than the value):
# bash tools/ab_prof.sh KNOB [VALUE]
knob=$1; val=${2:-1}
for v in 0 1; do
  if [ $v = 1 ]; then export $knob=$val; else unset $knob; fi
  python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$knob=' + ('$val' if $v else 'unset'), round(d['value']), {k:round(v['ms'],1) for k,v in d['kernels'].items()})"
done
