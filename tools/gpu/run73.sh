timeout 300 python tools/proj_time.py; FASTPFP_LIB=varlib/projold.so timeout 300 python tools/proj_time.py
for i in 1 2; do
timeout 300 python tools/prec_time.py c5 3 | tail -1
FASTPFP_LIB=varlib/projold.so timeout 300 python tools/prec_time.py c5 3 | tail -1
done
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
