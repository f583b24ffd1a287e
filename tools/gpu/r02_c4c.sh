# c4 A/B: new tile (two barriers per sweep) vs one barrier per sweep (per-lane column combine) vs the previous kernel
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/c4c_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c4c_tests.log
FASTPFP_LIB=varlib/var_onebar/libfastpfp.so timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/c4c_tests_onebar.log 2>&1; echo "tests onebar rc=$?"; tail -1 gpurun_out/c4c_tests_onebar.log
for rep in 1 2 3; do for v in "" varlib/var_onebar/libfastpfp.so varlib/var_ss_old/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 40 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
