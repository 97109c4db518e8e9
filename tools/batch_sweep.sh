python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "16384 2048" "32768 4096" "65536 4096" "65536 8192" "32768 8192"; do set -- $cfg
python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --max-tokens $1 --max-sents $2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['ms_per_step'],1), d['decode_steps'])"
done
