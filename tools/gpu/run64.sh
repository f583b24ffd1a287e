q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['value'], d['ms_per_step'], 'gemm', r['ms_per_launch'], 'proj', r['secondary']['ms_per_launch'], d['clocks'])"; }
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null | q cur
FASTPFP_LIB=varlib/merged.so timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null | q merged
done
