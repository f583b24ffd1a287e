for v in "" varlib/var_g4/libfastpfp.so varlib/var_g2/libfastpfp.so ""; do
  FASTPFP_LIB=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('lib=$v', d['value'], 'gemm', r['ms_per_launch'], 'proj', r['secondary']['ms_per_launch'], d['clocks']['sm_mhz'])"
done
for v in varlib/var_g4/libfastpfp.so varlib/var_g2/libfastpfp.so; do
  FASTPFP_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_i8 -c 2 python tools/ncu_driver.py c5 1 2>&1 | grep -E "dram__bytes|duration" | head -6
done
