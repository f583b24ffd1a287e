# c4: sigma from the row totals (16 fp32 adds per thread and sweep less)
timeout 900 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/g33_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g33_tests.log
for v in "" varlib/var_headD/libfastpfp.so "" varlib/var_headD/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
