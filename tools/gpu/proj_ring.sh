# c5 A/B: projection tiles issue their first bulk copies before loading the sum vectors (FPFP_PROJ_RING_FIRST) vs main
FASTPFP_LIB=varlib/var_ringfirst/libfastpfp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -x -q > gpurun_out/pr_tests.log 2>&1; echo "tests ringfirst rc=$?"; tail -1 gpurun_out/pr_tests.log
for rep in 1 2 3; do for v in "" varlib/var_ringfirst/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null > /tmp/c5.json
python -c "
import json,os; d=json.loads([l for l in open('/tmp/c5.json') if l.startswith('{')][-1]); r=d['roofline']; s=r.get('secondary',{})
print(os.environ.get('FASTPFP_LIB') or 'main', 'c5', d['value'], d['ms_per_step'], 'gemm ms', r['ms_per_launch'], 'proj ms', s.get('ms_per_launch'), 'proj frac', s.get('frac'), d['clocks']['sm_mhz'])"
done; done
