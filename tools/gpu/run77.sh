q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'])"; }
for i in 1 2; do
timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | q new
FASTPFP_LIB=varlib/ssprev.so timeout 600 python bench.py --workload c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | q prev
done
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity.py -x -q -k "batch or small or c4 or config4" 2>&1 | tail -2
