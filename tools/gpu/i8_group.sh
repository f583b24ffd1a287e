# c5 A/B under the power cap: int8 GEMM raster group of 4 / 16 M-tiles (FPFP_I8_GROUP) vs main (8);
# group 4 reads ~25 GB of DRAM per launch instead of ~36 GB (ncu), which may buy clock under sw_power_cap
for rep in 1 2 3; do for v in "" varlib/var_grp4/libfastpfp.so varlib/var_grp16/libfastpfp.so; do
export FASTPFP_LIB=$v
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-secondary --no-cpu-baseline 2>/dev/null > /tmp/c5.json
python -c "
import json,os; d=json.loads([l for l in open('/tmp/c5.json') if l.startswith('{')][-1]); r=d['roofline']; s=r.get('secondary',{})
print(os.environ.get('FASTPFP_LIB') or 'main', 'c5', d['value'], d['ms_per_step'], 'gemm ms', r['ms_per_launch'], 'proj ms', s.get('ms_per_launch'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
