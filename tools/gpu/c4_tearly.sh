# c4 A/B: t_i formed before the second slot barrier (FPFP_SS_T_EARLY) vs main
FASTPFP_LIB=varlib/var_tearly/libfastpfp.so timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/c4t_tests.log 2>&1; echo "tests tearly rc=$?"; tail -1 gpurun_out/c4t_tests.log
for rep in 1 2 3; do for v in "" varlib/var_tearly/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 40 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
