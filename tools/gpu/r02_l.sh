timeout 600 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -1
for v in "" varlib/var_tiles16/libfastpfp.so varlib/var_tiles32/libfastpfp.so ""; do
  FASTPFP_LIB=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('lib=$v', d['value'], 'gemm', r['ms_per_launch'], 'proj', r['secondary']['ms_per_launch'], r['secondary']['frac'], d['clocks']['sm_mhz'])"
done
