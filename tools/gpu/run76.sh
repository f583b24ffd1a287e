q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'])"; }
for i in 1 2; do
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | q default
FASTPFP_LIB=varlib/csum.so timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | q csum
done
FASTPFP_LIB=varlib/csum.so timeout 900 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -2
