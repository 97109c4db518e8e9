for cc in 0 1 0 1; do
python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --cap-clip $cc 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cap_clip=$cc', round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'steps', d['decode_steps'])"
done
for cc in 0 1; do
python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --cap-clip $cc --workers 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('W1 cap_clip=$cc', round(d['value']), 'ms/step', round(d['ms_per_step'],1), 'steps', d['decode_steps'])"
done
