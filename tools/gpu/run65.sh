for i in 1 2; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/sumstored.so timeout 300 python tools/prec_time.py c5 3 | tail -1
done
timeout 300 python tools/proj_time.py; FASTPFP_LIB=varlib/sumstored.so timeout 300 python tools/proj_time.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
