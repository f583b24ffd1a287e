for i in 1 2; do
timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new c4', d['value'], d['ms_per_step'])"
FASTPFP_LIB=varlib/ssold.so timeout 600 python bench.py --workload c4 --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('old c4', d['value'], d['ms_per_step'])"
done
