timeout 300 python -m pytest tests -m gpu -k "host" -x -q -p no:cacheprovider 2>&1 | tail -2
for CS in 1 2 3 4; do timeout 300 python bench.py --no-cpu --steps 6 --copy-streams $CS 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('copy_streams', $CS, 'e2e', round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))"; done
