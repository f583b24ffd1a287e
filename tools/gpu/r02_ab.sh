# c4: X loads of the blend through L1 (pass 2 re-reads pass 1's rows)
FASTPFP_LIB=varlib/var_xl1/libfastpfp.so timeout 600 python -m pytest tests/test_gpu_batched.py -x -q 2>&1 | tail -1
for v in "" varlib/var_xl1/libfastpfp.so "" varlib/var_xl1/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 300 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null > /tmp/c4.json
python -c "
import json,sys,os; d=json.loads([l for l in open('/tmp/c4.json') if l.startswith('{')][-1]); print(os.environ.get('FASTPFP_LIB') or 'main', 'c4', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
