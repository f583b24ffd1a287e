# checkpointed projection sweeps (replay): GPU suite, then c5 bench A/B (FPFP_PROJ_REPLAY=0 = previous kernel)
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/rp_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/rp_tests.log
python -m pytest tests/test_gpu_fullsize_lockstep.py -q -s -k sweep_sums 2>&1 | grep max_err_over_bound
for rep in 1 2; do for v in 1 0; do
export FPFP_PROJ_REPLAY=$v
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null > /tmp/c5.json
python -c "
import json,os; d=json.loads([l for l in open('/tmp/c5.json') if l.startswith('{')][-1]); r=d['roofline']; s=r.get('secondary',{})
print('replay', os.environ['FPFP_PROJ_REPLAY'], 'c5', d['value'], d['ms_per_step'], 'gemm ms', r['ms_per_launch'], 'proj ms', s.get('ms_per_launch'), 'proj frac', s.get('frac'), d['clocks']['sm_mhz'])"
done; done
unset FPFP_PROJ_REPLAY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:proj_kernel -c 1 -o gpurun_out/rp_proj -f python tools/ncu_driver.py c5 1 > gpurun_out/rp_ncu_proj.log 2>&1; echo "ncu proj rc=$?"
