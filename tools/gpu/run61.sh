timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'])"
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
