# bench value vs concurrent batch workers (GPU box), two rounds
for i in 1 2; do for w in 3 4 5 6; do
python bench.py --no-cpu-baseline --no-e2e --workers $w 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W=$w', round(d['value']), round(d['ms_per_step'],1))"
done; done
